cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_scale.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_scale.log 2>&1
echo done
