# Exchange variants on the visible GPUs: multi-GPU parity of every mode, then
# bench lines for the pass-along ring vs the one-hop all-gather (§8(f) row 3)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -5 > gpurun_out/pytest_multi.log
cat gpurun_out/pytest_multi.log
for mode in rma rma-ag sync; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29544 \
    bench.py --gpus $N --steps 20 --warmup 5 --mode $mode --staleness 0 --no-cpu-baseline > gpurun_out/bench_x_${mode}_s0.log 2>&1
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29544 \
    bench.py --gpus $N --steps 20 --warmup 5 --mode $mode --no-cpu-baseline > gpurun_out/bench_x_${mode}_s1.log 2>&1
done
for f in gpurun_out/bench_x_*.log; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], round(d['ms_per_step'],3), round(d['value']/1e6,1), 'Mev/s', {k: round(v,4) for k,v in d['phases_ms'].items() if k in ('exchange_adam_g',)}, d.get('exchange', {}))"; done
