# C5 convergence: async grouped ring vs synchronous all-reduce (4 GPUs), plus the grouped bench line
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555"
timeout 900 $R tests/tools/convergence.py --steps 600 --mode rma --group-size 2 --outer-every 10 --out gpurun_out/conv_rma_g2.json 2>&1 | grep -v Warning | tail -2
timeout 900 $R tests/tools/convergence.py --steps 600 --mode sync --out gpurun_out/conv_sync.json 2>&1 | grep -v Warning | tail -2
timeout 900 $R tests/tools/convergence.py --steps 600 --mode none --out gpurun_out/conv_none.json 2>&1 | grep -v Warning | tail -2
timeout 600 $R bench.py --gpus $N --steps 20 --warmup 3 --mode rma --group-size 2 --outer-every 10 > gpurun_out/bench_n${N}_rma_g2.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_n${N}_rma_g2.log').read().strip().splitlines()[-1]); print('grouped bench', d['n_gpus'], round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"
