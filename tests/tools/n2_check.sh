# 2-GPU: exchange timing per mode (paper packet and 201 MB), then the 2-GPU parity tests
tag=${1:-r02c}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29536 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for m in rma-ag rma-chunked rma; do
  timeout 300 $R --mode $m > gpurun_out/${tag}_n2_$m.jsonl 2> gpurun_out/${tag}_n2_$m.err
  timeout 300 $R --mode $m --gen-hidden 4096 > gpurun_out/${tag}_n2_${m}_big.jsonl 2> gpurun_out/${tag}_n2_${m}_big.err
done
timeout 900 python -m pytest tests/test_gpu_multi.py -q -k two 2>&1 | tail -3 > gpurun_out/${tag}_multi2.log
timeout 600 python -m pytest tests/test_gpu_exchange_emulated.py -q 2>&1 | tail -3 > gpurun_out/${tag}_emul.log
