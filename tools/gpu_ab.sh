set -x
mkdir -p gpurun_out/r10
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r10/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cluster or amg" > gpurun_out/r10/pytest_amg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r10/pytest_amg.log
B="timeout 600 python bench.py --no-cpu-baseline --no-variant"
VEM_AMG_UNROLL_NNZ=1e9 $B > gpurun_out/r10/U4.json 2> gpurun_out/r10/U4.err
$B > gpurun_out/r10/U8_l1.json 2> gpurun_out/r10/U8.err
VEM_AMG_UNROLL_NNZ=1e9 $B > gpurun_out/r10/U4b.json 2> gpurun_out/r10/U4b.err
$B > gpurun_out/r10/U8b_l1.json 2> gpurun_out/r10/U8b.err
