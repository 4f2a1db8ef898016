# A/B of lean-kernel variants (variant_<name>.so built at the repo root) on the
# default bench, then the parity tests on the last variant.
cd $GRAFT_REPO_ROOT
cp paper_2506_08781_b200/libposlo_gpu.so /tmp/base.so
rm -f gpurun_out/abo.txt
VARS=${VARS:-"base es base es"}
for v in $VARS; do
  if [ $v = base ]; then cp /tmp/base.so paper_2506_08781_b200/libposlo_gpu.so; else cp variant_$v.so paper_2506_08781_b200/libposlo_gpu.so; fi
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/abo_$v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/abo_$v.log').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['roofline']['ms_per_launch'], d['verdict'])" >> gpurun_out/abo.txt
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -p no:cacheprovider -x > gpurun_out/abo_tests.log 2>&1
