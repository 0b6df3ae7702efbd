# A/B of environment settings on the bench: ab_env.sh "VAR=a" "VAR=b" ...
# prints ms/step and the per-kernel table for each setting
mkdir -p gpurun_out
for setting in "$@"; do
  echo "=== $setting"
  env $setting timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>&1 || { tail -5 gpurun_out/ab.log; continue; }
  python - <<'PY'
import json
d = json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print(round(d['ms_per_step'], 3), {k: round(v, 3) for k, v in d['phases_ms'].items()})
for k, v in d['kernels']['per_kernel'].items():
    print(f"  {k:12s} {v['ms']:.3f} ms  hbm-floor {v['t_hbm_ms']:.3f}")
PY
done
