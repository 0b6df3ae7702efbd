# 2-GPU bench lines (default rma-ag and sync) with e2e host-input graph steps
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29537 bench.py --gpus 2"
for m in rma-ag sync rma; do
  timeout 400 $R --mode $m > gpurun_out/r02_n2e_$m.jsonl 2> gpurun_out/r02_n2e_$m.err
done
