# GPU call: the cluster-resident tridiagonalisation (k_trd_cluster) — tests, then c2 / c4 time to target A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_syev.py -m gpu -x -q > gpurun_out/c3_pytest_syev.log 2>&1; echo "rc=$?" >> gpurun_out/c3_pytest_syev.log
timeout 900 python -m pytest tests/test_gpu_cluster.py -m gpu -x -q > gpurun_out/c3_pytest_cluster.log 2>&1; echo "rc=$?" >> gpurun_out/c3_pytest_cluster.log
for cl in 1 0; do
  OZR_TRD_CLUSTER=$cl OZR_TRACE=1 timeout 300 python bench.py --config c2 --headline-only --no-cpu-baseline --e2e-steps 1 --steps 2 --warmup 1 > gpurun_out/c3_c2_cl$cl.log 2>&1
done
OZR_TRD_CLUSTER=1 OZR_TRACE=1 timeout 300 python tools/dev/syev_time.py 279 640 739 2734 6628 > gpurun_out/c3_syevtime_cl1.log 2>&1
OZR_TRD_CLUSTER=0 OZR_TRACE=1 timeout 300 python tools/dev/syev_time.py 279 640 739 2734 6628 > gpurun_out/c3_syevtime_cl0.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 2 --steps 5 --warmup 3 --no-c5 > gpurun_out/c3_bench_full.log 2>&1
