# Round-end evidence: bench lines for every config, the ncu launch list of the
# default bench, and one `ncu --set full` capture per hot kernel, exported to
# CSV (raw + source pages) so gpurun_out stays small.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python tools/pipe_probe.py > gpurun_out/pipe_probe.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json.log 2>&1
timeout 900 python bench.py --mode epoch --n2 1024 --log2n 30 --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/bench_c3.json.log 2>&1
timeout 900 python bench.py --varlen --mode epoch --n2 1024 --log2n 22 --steps 5 --warmup 3 --e2e-steps 2 --records > gpurun_out/bench_c4.json.log 2>&1
timeout 900 python bench.py --mode tamper --n2 1024 --log2n 30 --tamper 1024 --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/bench_c5.json.log 2>&1
timeout 600 python bench.py --suite 2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_s2.json.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
for spec in "k_hash_s1_l32r:--steps 3 --warmup 3" "k_check_thread16:--mode epoch --n2 1024 --log2n 28 --steps 1 --warmup 3" "k_hash_s1_var:--varlen --mode epoch --n2 1024 --log2n 22 --steps 1 --warmup 3" "k_hash_s2:--suite 2 --log2n 24 --steps 1 --warmup 3"; do
  k=${spec%%:*}; args=${spec#*:}
  POSLO_PIPE_PIECES=1 timeout 900 ncu --set full --clock-control none --import-source on -f -k regex:$k -c 1 -o /tmp/$k python bench.py $args --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  ncu -i /tmp/$k.ncu-rep --page raw --csv > gpurun_out/ncu_${k}_raw.csv 2>&1
  ncu -i /tmp/$k.ncu-rep --page source --csv > gpurun_out/ncu_${k}_source.csv 2>&1
done
du -sh gpurun_out
echo done
