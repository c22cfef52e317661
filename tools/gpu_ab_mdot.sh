set -x
R=r16
mkdir -p gpurun_out/$R
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/$R/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/$R/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$R/pytest_gpu.log
B="timeout 600 python bench.py --no-cpu-baseline --no-variant"
for i in 1 2 3; do
VEM_MDOT_WAVE=0 $B > gpurun_out/$R/wave0_$i.json 2> gpurun_out/$R/wave0_$i.err
VEM_MDOT_WAVE=1 $B > gpurun_out/$R/wave1_$i.json 2> gpurun_out/$R/wave1_$i.err
done
