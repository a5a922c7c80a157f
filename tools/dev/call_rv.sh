mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_refine.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/c2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c2_pytest.log
B="python bench.py --headline-only --no-cpu-baseline --e2e-steps 2 --steps 10 --warmup 3"
timeout 300 $B > gpurun_out/c2_bench_new.log 2>&1
OZR_RES_2PASS=1 timeout 300 $B > gpurun_out/c2_bench_2pass.log 2>&1
timeout 300 $B > gpurun_out/c2_bench_new2.log 2>&1
OZR_TRACE=1 timeout 300 python bench.py --config c2 --headline-only --no-cpu-baseline --e2e-steps 1 --steps 2 --warmup 1 > gpurun_out/c2_c2trace.log 2>&1
OZR_TRACE=1 OZR_SYEV_PROBE=1 timeout 300 python bench.py --config c2 --headline-only --no-cpu-baseline --e2e-steps 1 --steps 1 --warmup 1 > gpurun_out/c2_c2probe.log 2>&1
P="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 --headline-only"
timeout 600 ncu --set full --clock-control none -k regex:'k_recombine_V' -s 1 -c 2 -f -o gpurun_out/rV_full $P > gpurun_out/c2_ncu.log 2>&1
OZR_RES_2PASS=1 timeout 600 ncu --set full --clock-control none -k regex:'k_recombine_V' -s 1 -c 2 -f -o gpurun_out/rV_full_2pass $P > gpurun_out/c2_ncu2.log 2>&1
