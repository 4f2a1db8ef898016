cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x --deselect tests/test_gpu_dropin.py::test_reference_acceptance_on_both_drop_ins > gpurun_out/pytest_gpu.log 2>&1
python tools/step_breakdown.py > gpurun_out/step_breakdown.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_default.log 2>&1
echo done
