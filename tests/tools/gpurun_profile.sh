# One GPU-box pass: GPU tests, smoke, bench, ncu launch list, ncu --set full of the top kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
SAGIPS_TRACE=1 timeout 300 python tests/tools/trace_tc.py > gpurun_out/trace.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
# 6 k_bwd and 6 k_fwd launches per step (D: last, mid, first / first, mid, head; then G);
# step 3 (after 3 warm-up steps): k_bwd 18 = D backward of the last hidden layer, 20 = D backward of layer 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bwd -s 18 -c 3 -o gpurun_out/tc_bwd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bwd.log 2>&1
# k_fwd 18 = D first layer, 19 = middle, 20 = last hidden + head
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fwd -s 18 -c 3 -o gpurun_out/tc_fwd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_fwd.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sample -s 2 -c 1 -o gpurun_out/sample python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_sample.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
