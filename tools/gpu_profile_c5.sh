# ncu evidence for the C5 kind-5 path (each only after the plain run exited 0): the launch list of a
# bounded solve, summarised per kernel on the box (the raw csv is tens of MB), and one --set full
# capture per fine-level kernel reduced to its raw-metric CSV / details text (tools/gpu_ncu_c5.sh)
set -x
R=${1:-R2_27}
mkdir -p gpurun_out/$R
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/$R/build.log 2>&1
timeout 600 python tools/profile_step.py C5 2 5 > gpurun_out/$R/plain.log 2>&1 || exit 1
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80000 --csv --log-file /tmp/launches_c5.csv python tools/profile_step.py C5 2 5 > gpurun_out/$R/ncu_launch.log 2>&1
python tools/ncu_summary.py launches /tmp/launches_c5.csv gpurun_out/$R/launches_summary_c5.csv "C5 kind 5, 2 GMRES steps (1 K-PCG solve, 25 K steps), ncu gpu__time_duration per launch, no graphs" > gpurun_out/$R/summary.log 2>&1
bash tools/gpu_ncu_c5.sh $R
ls -la gpurun_out/$R
