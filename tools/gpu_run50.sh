cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/pipe_probe.py > gpurun_out/pipe_probe.log 2>&1
echo done
