timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/r02_par62.log
for g in 1 0 1 0; do SAGIPS_GEN_G=$g timeout 300 python bench.py --config c5 --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>&1; python - <<PY >> gpurun_out/r02_c5ab62.txt
import json
d = json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print("GEN_G=$g", round(d['ms_per_step'], 3), d['clocks']['sm_mhz'], " ".join(f"{k}={v['ms']:.3f}" for k, v in d['kernels']['per_kernel'].items()))
PY
done
