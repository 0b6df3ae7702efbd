# GPU tests + one bench line + trace (no profiling)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
SAGIPS_TRACE=1 timeout 300 python tests/tools/trace_tc.py > gpurun_out/trace.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print(round(d['ms_per_step'], 3), {k: round(v, 3) for k, v in d['phases_ms'].items()})
print('roofline', d['roofline']['kernel'], round(d['roofline']['achieved']), round(d['roofline']['frac'], 3))
for k, v in d['kernels']['per_kernel'].items():
    print(f"{k:12s} {v['ms']:.3f} ms {v['GBps']:6.0f} GB/s {v['TFLOPs']:6.1f} TF/s hbm-floor {v['t_hbm_ms']:.3f} tensor-floor {v['t_tensor_ms']:.3f}")
print(d["kernels"]["mlp_total"])
PY
