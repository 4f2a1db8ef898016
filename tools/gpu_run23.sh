cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 python bench.py --suite 2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_s2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hash_s1_l32r -c 1 -o /tmp/lean_full2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_ncu_full.log 2>&1
ncu -i /tmp/lean_full2.ncu-rep --page raw --csv > gpurun_out/lean_full2_raw.csv 2>&1
ncu -i /tmp/lean_full2.ncu-rep --page source --csv > gpurun_out/lean_full2_source.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_check_thread -c 1 -o /tmp/check_full python bench.py --mode epoch --n2 1024 --log2n 24 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_ncu_check.log 2>&1
ncu -i /tmp/check_full.ncu-rep --page raw --csv > gpurun_out/check_full_raw.csv 2>&1
ls -la gpurun_out > gpurun_out/ls.txt
du -sh gpurun_out >> gpurun_out/ls.txt
echo done
