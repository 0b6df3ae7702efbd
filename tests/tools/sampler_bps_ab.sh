for v in bps1 t1024 bps1 t1024; do
  if [ "$v" = base ]; then e=""; else e="SAGIPS_LIB_VARIANT=$v"; fi
  env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/sab.json').read().strip().splitlines()[-1])
print('$v', round(d['phases_ms']['sampler']*1e3,2), 'us in-step;', round(d['roofline_sampler_2p24']['us'],1), round(d['roofline_sampler_2p24_nohist']['us'],1), 'us 2^24 hist/nohist')" >> gpurun_out/r02_sab102.txt
done
