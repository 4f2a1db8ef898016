cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
oracle/_ref/test_distiller_gpu > gpurun_out/test_distiller_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/test_distiller_gpu.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo done
