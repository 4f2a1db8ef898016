cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/step_breakdown.py > gpurun_out/step_breakdown.log 2>&1
echo done
