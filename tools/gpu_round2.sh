# one round-2 GPU pass: build, GPU tests, smoke, bench (both arms), launch list
set -x
R=${1:-R2_01}
mkdir -p gpurun_out/$R
rm -f gpurun_out/parity_counts.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$R/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/$R/build.log 2>&1
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/$R/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$R/pytest_gpu.log
cp gpurun_out/parity_counts.jsonl gpurun_out/$R/parity_counts.jsonl
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$R/smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/$R/bench.json 2> gpurun_out/$R/bench.err
cp profiles/nested_counts.json gpurun_out/$R/nested_counts.json
tail -5 gpurun_out/$R/pytest_gpu.log; cat gpurun_out/$R/smoke.log | tail -5; head -c 3000 gpurun_out/$R/bench.json; tail -5 gpurun_out/$R/bench.err
