cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_epoch30.csv python bench.py --mode epoch --n2 1024 --log2n 30 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_ncu_e30.log 2>&1
echo done
