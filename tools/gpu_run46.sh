cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/scan_speed.py > gpurun_out/scan_speed.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_scan" -c 6 --csv python tools/scan_speed.py > gpurun_out/scan_ncu.csv 2>&1
echo done
