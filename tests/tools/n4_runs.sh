# 4-GPU: multi-process parity tests, then C4 (C2 per rank) bench lines per exchange mode
timeout 1200 python -m pytest tests/test_gpu_multi.py -q 2>&1 | tail -5 > gpurun_out/r02_pytest_multi_4gpu.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 4"
for m in rma-ag rma rma-chunked sync; do
  timeout 300 $R --mode $m > gpurun_out/r02_n4_$m.jsonl 2> gpurun_out/r02_n4_$m.err
done
timeout 300 $R --mode rma-ag --group-size 2 --outer-every 10 > gpurun_out/r02_n4_rma-ag_g2.jsonl 2> gpurun_out/r02_n4_rma-ag_g2.err
