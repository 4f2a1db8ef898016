cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 oracle/_ref/acceptance_gpu > gpurun_out/acceptance_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/acceptance_gpu.log
echo done
