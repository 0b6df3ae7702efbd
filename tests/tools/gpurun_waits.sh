# Per-role wait accounting of the layer passes: diagnostic rebuild with
# SAGIPS_BUILD_WAITS=1, then one traced step (tests/tools/trace_tc.py).
mkdir -p gpurun_out
SAGIPS_BUILD_WAITS=1 python paper_2407_00051_b200/build.py --force > gpurun_out/build_waits.log 2>&1
SAGIPS_TRACE=1 timeout 300 python tests/tools/trace_tc.py > gpurun_out/trace_waits.log 2>&1
cat gpurun_out/trace_waits.log
