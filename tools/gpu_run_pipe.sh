# A/B of the check pipelining for config 3 (2^30, 2^20 per-epoch checks):
# POSLO_PIPE_PIECES = 1 (hash all, then check), 4, 8 (default), 16.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for p in 1 4 8 16; do
  POSLO_PIPE_PIECES=$p timeout 900 python bench.py --mode epoch --n2 1024 --log2n 30 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3_p$p.json.log 2>&1
done
echo done
