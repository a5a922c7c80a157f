mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_syev.py -m gpu -x -q > gpurun_out/c6_pytest_syev.log 2>&1; echo "rc=$?" >> gpurun_out/c6_pytest_syev.log
OZR_SYEV_PROBE=1 OZR_TRACE=1 timeout 300 python tools/dev/syev_time.py 279 640 739 2734 > gpurun_out/c6_probe.log 2>&1
OZR_TRACE=1 timeout 300 python bench.py --config c2 --headline-only --no-cpu-baseline --e2e-steps 1 --steps 2 --warmup 1 > gpurun_out/c6_c2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_cluster.py -m gpu -x -q > gpurun_out/c6_pytest_cluster.log 2>&1; echo "rc=$?" >> gpurun_out/c6_pytest_cluster.log
