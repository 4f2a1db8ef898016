cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x --deselect tests/test_gpu_dropin.py::test_reference_acceptance_on_both_drop_ins > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --mode epoch --n2 1024 --log2n 26 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_e26.log 2>&1
timeout 900 python bench.py --mode epoch --n2 1024 --log2n 30 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_e30.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_check|k_decode|k_table|k_fold|k_segfold" -c 30 --csv python bench.py --mode epoch --n2 1024 --log2n 28 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/fe_launches.csv 2>&1
python tools/step_breakdown.py > gpurun_out/step_breakdown.log 2>&1
echo done
