# ncu evidence for the C5 kind-5 path: launch list of a bounded solve, one --set full capture
# of the fine-level kernels, then times of the other configs (each only after the plain run)
set -x
R=${1:-R2_03}
mkdir -p gpurun_out/$R
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/$R/build.log 2>&1
timeout 600 python tools/profile_step.py C5 2 5 > gpurun_out/$R/plain.log 2>&1 || exit 1
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80000 --csv --log-file gpurun_out/$R/launches.csv python tools/profile_step.py C5 2 5 > gpurun_out/$R/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_seps_resid|k_pcg_spmv_p|k_mg_blk|k_kmul|k_br_finish|k_vc_cheb_step|k_pcgm_xr' -s 60 -c 21 -o gpurun_out/$R/full python tools/profile_step.py C5 2 5 > gpurun_out/$R/ncu_full.log 2>&1
timeout 900 python tools/run_configs.py C1,C2,C4,C2:5,C4:5 5000 > gpurun_out/$R/configs.jsonl 2> gpurun_out/$R/configs.err
ls -la gpurun_out/$R
cut -c 1-420 gpurun_out/$R/configs.jsonl
