set -x
mkdir -p gpurun_out/r6
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r6/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r6/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r6/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r6/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r6/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r6/bench.json 2> gpurun_out/r6/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r6/reference.json 2> gpurun_out/r6/reference.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/r6/launches.csv python tools/profile_step.py C3 20000 3 > gpurun_out/r6/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_vc_cheb_step|k_vc_cheb_first|k_vc_spmv_z|k_vc_sa_|k_vc_resid|k_mdot|k_update' -s 40 -c 16 -o gpurun_out/r6/full python tools/profile_step.py C3 30 3 > gpurun_out/r6/ncu_full.log 2>&1
ls -la gpurun_out/r6
