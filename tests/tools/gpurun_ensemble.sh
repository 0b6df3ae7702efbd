# Ensemble analysis vs training time on the visible GPUs (tests/tools/ensemble.py):
#   gpurun_ensemble.sh STEPS EVERY TAG
STEPS=${1:-100000}; EVERY=${2:-5000}; TAG=${3:-r01}
mkdir -p gpurun_out/ensemble
N=$(nvidia-smi -L | wc -l)
run() {  # name args...
  local name=$1; shift
  timeout 3000 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29561 tests/tools/ensemble.py --steps $STEPS --every $EVERY "$@" \
    --out gpurun_out/ensemble/${TAG}_${name}_n${N}.json > gpurun_out/ensemble/${TAG}_${name}_n${N}.log 2>&1
  tail -1 gpurun_out/ensemble/${TAG}_${name}_n${N}.log
}
run none --mode none --seed-per-rank
run rma_split --mode rma --group-size 2 --split-batch
run rma_full --mode rma --group-size 2
