# sweep the pipelined step's CTAs-per-role split (SAGIPS_PIPE_SPLIT_D/_G)
for sd in "27,15,28,26,26,26" "24,24,26,25,25,24" "22,28,26,24,24,24" "20,32,26,24,24,22" "18,36,26,24,24,20"; do
  SAGIPS_PIPE_SPLIT_D=$sd timeout 120 python bench.py --no-cpu-baseline --no-e2e --steps 6 --warmup 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('D $sd', round(d['phases_ms']['disc_step'],3), 'G', round(d['phases_ms']['gen_loss_through_disc'],3))"
done
for sg in "38,20,37,17,17,19" "30,30,34,18,18,18" "26,36,34,18,18,16" "24,40,32,18,18,16"; do
  SAGIPS_PIPE_SPLIT_G=$sg timeout 120 python bench.py --no-cpu-baseline --no-e2e --steps 6 --warmup 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('G $sg', round(d['phases_ms']['gen_loss_through_disc'],3))"
done
