# CTA timelines of the D backward passes with and without the G_4 regeneration (kGenG)
mkdir -p gpurun_out
for g in 1 0; do SAGIPS_GEN_G=$g SAGIPS_TRACE=1 timeout 300 python tests/tools/trace_tc.py > gpurun_out/r02_trace48_g$g.log 2>&1; done
