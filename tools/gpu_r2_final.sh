#!/bin/bash
# Round-2 evidence on one B200: smoke, the whole GPU suite, bench lines for
# every config (default = config 2 with e2e / drop-in / cpu_baseline; the
# reference arm; configs 3, 4, 5, suite 2), the ncu launch list of the default
# bench, and ncu --set full captures (raw + per-SASS source pages) of the hot
# kernels at the BASELINE per-GPU sizes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/final
O=gpurun_out/final
T="timeout -k 20"
$T 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
$T 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
tail -2 $O/pytest_gpu.log
$T 300 python tools/pipe_probe.py > $O/pipe_probe.log 2>&1
$T 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
$T 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
$T 900 python bench.py --mode epoch --n2 1024 --log2n 30 --steps 3 --warmup 3 --e2e-steps 0 > $O/bench_c3.json 2> $O/bench_c3.err
$T 900 python bench.py --varlen --mode epoch --n2 1024 --log2n 25 --steps 3 --warmup 3 --e2e-steps 1 > $O/bench_c4_share.json 2> $O/bench_c4_share.err
POSLO_PIPE_PIECES=1 $T 900 python bench.py --varlen --mode epoch --n2 1024 --log2n 25 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/bench_c4_share_p1.json 2> $O/bench_c4_share_p1.err
$T 900 python bench.py --varlen --mode epoch --n2 1024 --log2n 22 --steps 5 --warmup 3 --e2e-steps 2 --records > $O/bench_c4.json 2> $O/bench_c4.err
$T 900 python bench.py --mode tamper --n2 1024 --log2n 30 --tamper 1024 --steps 3 --warmup 3 --e2e-steps 0 > $O/bench_c5.json 2> $O/bench_c5.err
$T 600 python bench.py --suite 2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_s2.json 2> $O/bench_s2.err
$T 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-dropin > /dev/null 2>&1
for spec in "k_hash_s1_l32r:--steps 3 --warmup 3" "k_hash_s1_var:--varlen --mode epoch --n2 1024 --log2n 25 --steps 1 --warmup 3" "k_check16e_comb:--mode epoch --n2 1024 --log2n 28 --steps 1 --warmup 3" "k_batch_invert:--mode epoch --n2 1024 --log2n 28 --steps 1 --warmup 3"; do
  k=${spec%%:*}; args=${spec#*:}
  POSLO_PIPE_PIECES=1 $T 1200 ncu --set full --clock-control none --import-source on -f -k regex:$k -c 1 -o /tmp/$k python bench.py $args --no-cpu-baseline --e2e-steps 0 --no-dropin > /dev/null 2>&1
  ncu -i /tmp/$k.ncu-rep --page raw --csv > $O/ncu_${k}_raw.csv 2>&1
  ncu -i /tmp/$k.ncu-rep --page source --csv --print-source sass > $O/ncu_${k}_sass.csv 2>&1
done
du -sh gpurun_out
echo done
