# 4-GPU measurement recipe (DESIGN §9, §8(f) row 3): the synchronous
# all-reduce under each NCCL algorithm for the library's communicators
# (bench.py --nccl-algo), the one-sided ring and the one-hop all-gather at
# staleness 0.
mkdir -p gpurun_out/nccl
run4() { timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NP:-4} --master-addr 127.0.0.1 --master-port $1 bench.py --gpus ${NP:-4} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "${@:2}"; }
for algo in default NVLS Ring Tree; do
  extra=""; [ $algo != default ] && extra="--nccl-algo $algo"
  NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING run4 29542 --mode sync --staleness 0 $extra > gpurun_out/nccl/sync_$algo.out 2> gpurun_out/nccl/sync_$algo.err
  echo "sync $algo rc=$?"; grep '^{' gpurun_out/nccl/sync_$algo.out > gpurun_out/nccl/sync_$algo.jsonl
done
for m in rma rma-ag; do
  run4 29543 --mode $m --staleness 0 > gpurun_out/nccl/${m}_s0.jsonl 2> gpurun_out/nccl/${m}_s0.err; echo "$m s0 rc=$?"
done
