# multi-GPU: exchange parity tests + weak-scaling bench lines for N = 1, 2, ..., visible GPUs
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -5 > gpurun_out/pytest_multi.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n1.log 2>&1
for n in 2 4 8; do
  [ $n -le $N ] || continue
  for mode in rma sync; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29544 \
      bench.py --gpus $n --steps 10 --warmup 3 --mode $mode > gpurun_out/bench_n${n}_${mode}.log 2>&1
  done
  if [ $n -ge 4 ]; then
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29544 \
      bench.py --gpus $n --steps 10 --warmup 3 --mode rma --group-size 2 --outer-every 10 > gpurun_out/bench_n${n}_rma_g2.log 2>&1
  fi
done
cat gpurun_out/pytest_multi.log
for f in gpurun_out/bench_n*.log; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], round(d['ms_per_step'],3), round(d['value']/1e6,1), 'Mev/s', d['config'].get('workload')[-40:], {k: round(v,3) for k,v in d['phases_ms'].items() if k in ('disc_step','exchange_adam_g')}, {k: round(v,2) for k,v in (d.get('exchange') or {}).items() if k in ('us_min_over_ranks','us_max_over_ranks','achieved')})"; done
