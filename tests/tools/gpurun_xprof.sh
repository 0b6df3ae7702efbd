# exchange kernel durations (torch.profiler) under push-CTA / fence variants
for v in "SAGIPS_PUSH_CTAS=1" "SAGIPS_PUSH_CTAS=8" "SAGIPS_PUSH_CTAS=32" "SAGIPS_PUSH_CTAS=148" "SAGIPS_PUSH_CTAS=32 SAGIPS_PUSH_NOFENCE=1"; do
  echo "== $v"
  env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29545 tests/tools/xprof.py --mode rma 2>&1 | grep -A2 "^rank 0"
done
