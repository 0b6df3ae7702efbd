# k_push time vs packet size at N = 2 (the ~9 us floor of the paper-size push): generator widths 8 .. 1024
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29539 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --mode rma-ag"
for h in 8 32 128 512 1024; do
  timeout 300 $R --gen-hidden $h > gpurun_out/pf.json 2>/dev/null
  python - <<PY >> gpurun_out/r02_push_floor.txt
import json
d = json.loads(open('gpurun_out/pf.json').read().strip().splitlines()[-1])
x = d['exchange']
print(f"gen_hidden $h packet {x['packet_bytes']:>10d} B  push {x['push_us']:8.2f} us  exchange {x['us_min_over_ranks']:8.2f} us")
PY
done
