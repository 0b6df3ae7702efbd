# Same-box A/B of library builds: ab_lib.sh VARIANT... runs the bench with
# libsagips.so ("base") and each paper_2407_00051_b200/libsagips_VARIANT.so,
# twice each, interleaved; prints ms/step and the per-kernel table
mkdir -p gpurun_out
for rep in 1 2; do
  for v in base "$@"; do
    echo "=== $v (run $rep)"
    if [ "$v" = base ]; then e=""; else e="SAGIPS_LIB_VARIANT=$v"; fi
    env $e timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>&1 || { tail -5 gpurun_out/ab.log; continue; }
    python - <<'PY'
import json
d = json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print(round(d['ms_per_step'], 3), " ".join(f"{k}={v['ms']:.4f}" for k, v in d['kernels']['per_kernel'].items()))
PY
  done
done
