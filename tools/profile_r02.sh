#!/bin/bash
# Round-2 ncu captures (run on the GPU box via gpurun; one GPU).  Each ncu run
# follows the same command's plain run (exit 0) per B200_PROFILING.md.
set -u
O=gpurun_out
C5="python tools/solve_once.py --config 5 --reps 1 --iters 4"
C4="python tools/solve_once.py --config 4 --reps 1 --iters 6"
$C5 > $O/c5_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 2 -c 1 \
      -o $O/r02_umma_c5 $C5 > $O/c5_ncu.log 2>&1
$C5 > $O/c5_plain2.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/r02_launches_c5.csv $C5 > $O/c5_launch.log 2>&1
$C4 > $O/c4_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fused_ps -s 3 -c 1 \
      -o $O/r02_fused_c4 $C4 > $O/c4_ncu.log 2>&1
$C4 > $O/c4_plain2.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/r02_launches_c4.csv $C4 > $O/c4_launch.log 2>&1
tail -2 $O/*_ncu.log $O/*_launch.log
