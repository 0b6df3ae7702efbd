# C2 (fp32-class, 2^20 events per rank) convergence on 4 GPUs with the final kernels: async one-hop all-gather
# (s = 1), grouped (g = 2, outer every 10), synchronous all-reduce, independent GANs
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 tests/tools/convergence.py --steps 2000 --every 100 --events-per-sample 1024 --precision fp32"
mkdir -p gpurun_out/conv_c2
timeout 600 $R --mode rma-ag --out gpurun_out/conv_c2/rma-ag.json > gpurun_out/conv_c2/rma-ag.txt 2>&1
timeout 600 $R --mode rma-ag --group-size 2 --outer-every 10 --out gpurun_out/conv_c2/rma-ag_g2.json > gpurun_out/conv_c2/rma-ag_g2.txt 2>&1
timeout 600 $R --mode sync --out gpurun_out/conv_c2/sync.json > gpurun_out/conv_c2/sync.txt 2>&1
timeout 600 $R --mode none --out gpurun_out/conv_c2/none.json > gpurun_out/conv_c2/none.txt 2>&1
