cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/step_breakdown.py > gpurun_out/step_breakdown.log 2>&1
python tools/step_breakdown.py >> gpurun_out/step_breakdown.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_seed" -c 5 --csv python tools/step_breakdown.py > gpurun_out/k0.csv 2>&1
echo done
