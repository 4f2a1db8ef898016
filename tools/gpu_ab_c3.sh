cd $GRAFT_REPO_ROOT
cp paper_2506_08781_b200/libposlo_gpu.so /tmp/base.so
rm -f gpurun_out/abc3.txt
for v in base e4 base e4; do
  if [ $v = base ]; then cp /tmp/base.so paper_2506_08781_b200/libposlo_gpu.so; else cp variant_$v.so paper_2506_08781_b200/libposlo_gpu.so; fi
  python bench.py --mode epoch --n2 1024 --log2n 28 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/abc3_$v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/abc3_$v.log').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['roofline']['ms_per_launch'], d['verdict'])" >> gpurun_out/abc3.txt
done
cp /tmp/base.so paper_2506_08781_b200/libposlo_gpu.so
python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_distill.py tests/test_gpu_signer.py -q -p no:cacheprovider -x > gpurun_out/abc3_tests.log 2>&1
