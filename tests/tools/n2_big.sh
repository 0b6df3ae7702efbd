# 2-GPU large-packet exchange (generator hidden 4096: 201 MB packets), one line per mode
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 10 --warmup 3"
tag=${1:-r2}
for m in rma-ag rma-chunked sync; do
  timeout 300 $R --mode $m --gen-hidden 4096 > gpurun_out/${tag}_n2_${m}_big.jsonl 2> gpurun_out/${tag}_n2_${m}_big.err
done
