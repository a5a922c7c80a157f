mkdir -p gpurun_out
OZR_SYEV_PROBE=1 OZR_TRACE=1 timeout 300 python tools/dev/syev_time.py 279 640 739 > gpurun_out/c5_probe.log 2>&1
