R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3"
for m in rma-ag rma-chunked rma sync; do
  timeout 300 $R --mode $m > gpurun_out/r2_n2b_$m.jsonl 2> gpurun_out/r2_n2b_$m.err
  timeout 300 $R --mode $m --gen-hidden 4096 > gpurun_out/r2_n2b_${m}_big.jsonl 2> gpurun_out/r2_n2b_${m}_big.err
done
timeout 900 python -m pytest tests/test_gpu_multi.py -q -k two 2>&1 | tail -5 > gpurun_out/r2_multi2b.log
