cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x --deselect tests/test_gpu_dropin.py::test_reference_acceptance_on_both_drop_ins > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --mode tamper --n2 1024 --log2n 26 --tamper 16 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_t26.log 2>&1
timeout 900 python bench.py --mode tamper --n2 1024 --log2n 30 --tamper 1024 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_t30.log 2>&1
echo done
