# Varlen (config 4) iteration: parity tests on the varlen / pipelined paths, a
# config-4 bench line, and one ncu --set full capture of k_hash_s1_var.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_logfile.py -q -p no:cacheprovider -k "length or ragged or varlen or chunked or log or large" > gpurun_out/var_tests.log 2>&1
timeout 600 python bench.py --varlen --mode epoch --n2 1024 --log2n 22 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c4_v3.json.log 2>&1
timeout 900 python bench.py --mode epoch --n2 1024 --log2n 30 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3_v3.json.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_s1_var -c 1 -o /tmp/kv python bench.py --varlen --mode epoch --n2 1024 --log2n 22 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu -i /tmp/kv.ncu-rep --page raw --csv > gpurun_out/ncu_var_v3_raw.csv 2>&1
ncu -i /tmp/kv.ncu-rep --page source --csv > gpurun_out/ncu_var_v3_source.csv 2>&1
echo done
