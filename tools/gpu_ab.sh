set -x
mkdir -p gpurun_out/r14
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r14/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "amg or cluster" > gpurun_out/r14/pytest_amg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r14/pytest_amg.log
B="timeout 600 python bench.py --no-cpu-baseline --no-variant"
for i in 1 2 3; do
VEM_PDL=0 $B > gpurun_out/r14/pdl0_$i.json 2> gpurun_out/r14/pdl0_$i.err
VEM_PDL=1 $B > gpurun_out/r14/pdl1_$i.json 2> gpurun_out/r14/pdl1_$i.err
done
