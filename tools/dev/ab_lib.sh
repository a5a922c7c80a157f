# A/B of two libozr.so builds on one box: paper_2602_19090_b200/libozr.so (new) vs libozr_old.so (old):
# quick GPU parity, alternating bench runs, and the launch list of each at the locked base clock.
set -x
cd $GRAFT_REPO_ROOT
P=paper_2602_19090_b200
cp $P/libozr.so /tmp/libozr_new.so
cp $P/libozr_old.so /tmp/libozr_old.so
timeout 900 python -m pytest tests/test_gpu_refine.py tests/test_gpu_split.py -x -q -m gpu > gpurun_out/ab_tests.log 2>&1; tail -3 gpurun_out/ab_tests.log
for v in new old new old; do
  cp /tmp/libozr_$v.so $P/libozr.so
  timeout 300 python bench.py --steps 10 --warmup 3 --no-c4 --no-cpu-baseline > gpurun_out/ab_bench_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_bench_$v.json'));print('$v',d['ms_per_step'],d['value'],d['clocks'])"
done
for v in new old; do
  cp /tmp/libozr_$v.so $P/libozr.so
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control base -k regex:'^k_' --csv --log-file gpurun_out/ab_launch_$v.csv python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-c4 --no-cpu-baseline > /dev/null 2>&1
done
cp /tmp/libozr_new.so $P/libozr.so
