# A/B of variable-length kernel variants (variant_<name>.so at the repo root)
# on config 4, then the varlen parity tests on the last variant.
cd $GRAFT_REPO_ROOT
cp paper_2506_08781_b200/libposlo_gpu.so /tmp/base.so
rm -f gpurun_out/abv.txt
VARS=${VARS:-"base v3 base v3"}
for v in $VARS; do
  if [ $v = base ]; then cp /tmp/base.so paper_2506_08781_b200/libposlo_gpu.so; else cp variant_$v.so paper_2506_08781_b200/libposlo_gpu.so; fi
  python bench.py --varlen --mode epoch --n2 1024 --log2n 22 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/abv_$v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/abv_$v.log').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['roofline']['ms_per_launch'], d['verdict'])" >> gpurun_out/abv.txt
done
python -m pytest tests/test_gpu_parity.py tests/test_logfile.py -q -p no:cacheprovider -x -k "length or ragged or varlen or log" > gpurun_out/abv_tests.log 2>&1
