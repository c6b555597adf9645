#!/bin/bash
# Round-2 ncu captures of the remaining configs' dominant kernels (configs 1-3;
# configs 4 and 5: tools/profile_r02.sh).  One GPU; each ncu run follows the
# same command's plain run (exit 0) per B200_PROFILING.md.  The reports are
# exported to CSV (raw page + SASS source page) on the box and deleted, so
# gpurun_out/ stays under the copy-back limit.
set -u
O=gpurun_out
C1="python tools/solve_once.py --config 1 --reps 1"
C2="python tools/solve_once.py --config 2 --reps 1 --iters 12"
C3="python tools/solve_once.py --config 3 --reps 1 --iters 6"
export_rep() {
  ncu -i "$1.ncu-rep" --page raw --csv > "$1.raw.csv" 2>/dev/null
  ncu -i "$1.ncu-rep" --page source --csv --print-source sass > "$1.src.csv" 2>/dev/null
  rm -f "$1.ncu-rep"
}
$C2 > $O/c2_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fgemm_pass -s 3 -c 1 \
      -o $O/r02_fgemm_c2 $C2 > $O/c2_ncu.log 2>&1 && export_rep $O/r02_fgemm_c2
$C2 > $O/c2_plain2.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/r02_launches_c2.csv $C2 > $O/c2_launch.log 2>&1
$C3 > $O/c3_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sep_sweep -s 3 -c 1 \
      -o $O/r02_sep_c3 $C3 > $O/c3_ncu.log 2>&1 && export_rep $O/r02_sep_c3
$C3 > $O/c3_plain2.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/r02_launches_c3.csv $C3 > $O/c3_launch.log 2>&1
$C1 > $O/c1_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:small_solve -c 1 \
      -o $O/r02_small_c1 $C1 > $O/c1_ncu.log 2>&1 && export_rep $O/r02_small_c1
for f in $O/c*_ncu.log $O/c*_launch.log; do echo "== $f"; tail -n 2 "$f"; done
du -sh $O
