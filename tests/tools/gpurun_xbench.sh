mkdir -p gpurun_out
for mode in rma rma-ag arar sync; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 \
  bench.py --gpus 2 --steps 20 --warmup 5 --mode $mode --no-cpu-baseline > gpurun_out/xb_$mode.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/xb_$mode.log').read().strip().splitlines()[-1]); print('$mode', round(d['ms_per_step'],3), d['exchange'])" || tail -5 gpurun_out/xb_$mode.log
done
