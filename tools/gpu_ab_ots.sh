cd $GRAFT_REPO_ROOT
cp paper_2506_08781_b200/libposlo_gpu.so /tmp/base.so
rm -f gpurun_out/abo.txt
for v in base ots ots5 base ots ots5; do
  if [ $v = base ]; then cp /tmp/base.so paper_2506_08781_b200/libposlo_gpu.so; else cp variant_$v.so paper_2506_08781_b200/libposlo_gpu.so; fi
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/abo_$v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/abo_$v.log').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['roofline']['ms_per_launch'], d['verdict'])" >> gpurun_out/abo.txt
done
cp variant_ots5.so paper_2506_08781_b200/libposlo_gpu.so
python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "uniform or golden or ekeys or paver or verdicts" > gpurun_out/abo_tests.log 2>&1
