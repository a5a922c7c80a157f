#!/bin/bash
# Round profile capture (run on the GPU box from the repo root, under gpurun). Outputs in gpurun_out/.
#   1. launch list of the library's kernels over one bench invocation (cold-cache, serialised)
#   2. one `ncu --set full` capture of the slice GEMM (the V product of the 2nd sweep)
#   3. one `ncu --set full` capture of each HBM-bound kernel of the 2nd sweep
set -x
OUT=gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 --headline-only"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' --csv --log-file $OUT/launches.csv $B > $OUT/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemm_i8 -s 3 -c 1 -f -o $OUT/gemm_full $B > $OUT/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_x1_split|k_recombine_V|k_split_fixed|k_split_res|k_recombine_E|k_final|k_transpose_i8' -s 8 -c 8 -f -o $OUT/hbm_full $B > $OUT/ncu_hbm.log 2>&1
