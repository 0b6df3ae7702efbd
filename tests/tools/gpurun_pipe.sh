# GPU tests, then pipelined vs per-layer step: bench lines + traces
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/bench_pipe.log 2>&1
SAGIPS_PIPE=0 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/bench_layers.log 2>&1
SAGIPS_TRACE=1 timeout 300 python tests/tools/trace_tc.py > gpurun_out/trace_pipe.log 2>&1
SAGIPS_PIPE=0 SAGIPS_TRACE=1 timeout 300 python tests/tools/trace_tc.py > gpurun_out/trace_layers.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for f in gpurun_out/bench_pipe.log gpurun_out/bench_layers.log; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
cat gpurun_out/trace_pipe.log gpurun_out/trace_layers.log
