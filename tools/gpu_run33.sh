cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_default.log 2>&1
timeout 900 python bench.py --mode epoch --n2 1024 --log2n 26 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_epoch26.log 2>&1
timeout 900 python bench.py --mode tamper --n2 1024 --log2n 26 --tamper 16 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_tamper26.log 2>&1
timeout 900 python bench.py --varlen --mode epoch --n2 1024 --log2n 22 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_var22.log 2>&1
POSLO_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --log2n 22 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/bench_w2_gloo.log 2>&1
echo done
