# sweep the pipelined step's CTAs-per-role split (SAGIPS_PIPE_SPLIT_D/_G)
for sd in "25,21,25,25,26,26" "24,22,24,26,26,26" "22,22,26,26,26,26" "26,20,26,25,25,26"; do
  SAGIPS_PIPE=1 SAGIPS_PIPE_SPLIT_D=$sd timeout 120 python bench.py --no-cpu-baseline --no-e2e --steps 6 --warmup 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('D $sd', round(d['phases_ms']['disc_step'],3), 'G', round(d['phases_ms']['gen_loss_through_disc'],3))"
done
for sg in "34,26,26,24,23,15" "32,26,28,24,24,14" "30,28,28,24,24,14"; do
  SAGIPS_PIPE=1 SAGIPS_PIPE_SPLIT_G=$sg timeout 120 python bench.py --no-cpu-baseline --no-e2e --steps 6 --warmup 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('G $sg', round(d['phases_ms']['gen_loss_through_disc'],3))"
done
