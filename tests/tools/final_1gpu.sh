# Round-end evidence on one GPU: the GPU test suite, smoke(), and the bench lines (C2 / C1 / C5 / reference arm)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r02_final_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_final_smoke.log 2>&1
for c in c2 c1 c5; do timeout 500 python bench.py --config $c > gpurun_out/r02_final_bench_$c.jsonl 2> gpurun_out/r02_final_bench_$c.err; done
timeout 400 python bench.py --impl reference > gpurun_out/r02_final_bench_reference.jsonl 2> gpurun_out/r02_final_bench_reference.err
