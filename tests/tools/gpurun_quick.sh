# GPU tests + one bench line (no profiling)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
SAGIPS_TRACE=1 timeout 300 python tests/tools/trace_tc.py > gpurun_out/trace.log 2>&1
tail -5 gpurun_out/pytest_gpu.log; tail -c 1500 gpurun_out/bench.log
