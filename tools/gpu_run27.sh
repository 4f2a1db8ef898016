cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for t in 1024 512 256; do
POSLO_VAR_TILE=$t timeout 900 python bench.py --varlen --mode epoch --n2 1024 --log2n 22 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_var22_t$t.log 2>&1
done
POSLO_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --log2n 22 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/bench_w2_gloo.log 2>&1
POSLO_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --mode tamper --n2 1024 --log2n 22 --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/bench_w2_tamper_gloo.log 2>&1
echo done
