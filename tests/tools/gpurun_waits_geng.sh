mkdir -p gpurun_out
timeout 300 bash tests/tools/ab_env.sh "SAGIPS_GEN_G=1" "SAGIPS_GEN_G=0" > gpurun_out/r02_ab47.txt 2>&1
SAGIPS_BUILD_WAITS=1 python paper_2407_00051_b200/build.py --force > gpurun_out/build_waits.log 2>&1
for g in 1 0; do SAGIPS_GEN_G=$g SAGIPS_TRACE=1 timeout 300 python tests/tools/trace_tc.py > gpurun_out/r02_waits47_g$g.log 2>&1; done
