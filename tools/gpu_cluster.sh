set -x
mkdir -p gpurun_out/r7c
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r7c/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cluster or amg" > gpurun_out/r7c/pytest_amg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r7c/pytest_amg.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r7c/bench.json 2> gpurun_out/r7c/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/r7c/launches.csv python tools/profile_step.py C3 20000 3 > gpurun_out/r7c/ncu_launch.log 2>&1
