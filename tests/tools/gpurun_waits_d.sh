# per-role wait accounting of the D backward passes (diagnostic rebuild), default settings
mkdir -p gpurun_out
SAGIPS_BUILD_WAITS=1 python paper_2407_00051_b200/build.py --force > gpurun_out/build_waits.log 2>&1
SAGIPS_TRACE=1 timeout 300 python tests/tools/trace_tc.py > gpurun_out/${1:-r02}_waits_d.log 2>&1
