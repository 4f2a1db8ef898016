cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
for m in 0 1 2; do
  POSLO_SHA_MODE=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_mode$m.log 2>&1
done
python - > gpurun_out/microbench.log 2>&1 <<'PY'
import ctypes
lib = ctypes.CDLL("paper_2506_08781_b200/libposlo_microbench.so")
lib.poslo_microbench_int_peak.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
for mode in (0, 1, 2, 0, 1, 2):
    v, ms = ctypes.c_double(), ctypes.c_double()
    lib.poslo_microbench_int_peak(0, mode, ctypes.byref(v), ctypes.byref(ms))
    print(mode, v.value / 1e12, ms.value)
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hash_s1 -s 2 -c 1 -o gpurun_out/prof_hash_s1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1
echo done
