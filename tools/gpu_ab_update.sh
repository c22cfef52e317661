set -x
R=r17
mkdir -p gpurun_out/$R
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/$R/build.log 2>&1
B="timeout 600 python bench.py --no-cpu-baseline --no-variant"
for i in 1 2 3; do
VEM_UPDATE_WAVE=0 $B > gpurun_out/$R/uwave0_$i.json 2> gpurun_out/$R/uwave0_$i.err
VEM_UPDATE_WAVE=1 $B > gpurun_out/$R/uwave1_$i.json 2> gpurun_out/$R/uwave1_$i.err
done
VEM_UPDATE_WAVE=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/$R/pytest_gpu_uwave1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$R/pytest_gpu_uwave1.log
