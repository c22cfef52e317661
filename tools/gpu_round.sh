set -x
R=${1:-r6}
mkdir -p gpurun_out/$R
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$R/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/$R/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/$R/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$R/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$R/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/$R/bench.json 2> gpurun_out/$R/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/$R/reference.json 2> gpurun_out/$R/reference.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/$R/launches.csv python tools/profile_step.py C3 20000 3 > gpurun_out/$R/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_vc_cheb_step|k_vc_cheb_first|k_vc_spmv_z|k_vc_sa_|k_vc_resid|k_mdot|k_update' -s 40 -c 16 -o gpurun_out/$R/full python tools/profile_step.py C3 30 3 > gpurun_out/$R/ncu_full.log 2>&1
ls -la gpurun_out/$R
timeout 900 python tools/run_configs.py C1,C2,C3,C4 5000 > gpurun_out/$R/configs.jsonl 2> gpurun_out/$R/configs.err
timeout 900 python tools/kernel_roofline.py C5:2:20 C4:1:100 C4:2:50 C2:1:210 > gpurun_out/$R/kernel_roofline.jsonl 2> gpurun_out/$R/kernel_roofline.err
ls -la gpurun_out/$R
