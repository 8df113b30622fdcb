#!/bin/bash
# GPU box: one `ncu --set full` capture of the first launch of each named kernel in
# one sq_sort_u32 of cfg5 (after the same command ran clean without ncu).  The
# reports are summarised on the box (metrics table, per-source-line hot spots);
# set KEEP=1 to bring the .ncu-rep back too (gpurun returns at most 64 MiB).
set -u
mkdir -p gpurun_out
timeout 120 python tools/sort_once.py > gpurun_out/sort_once.log 2>&1 || exit 1
for k in "$@"; do
  rep=gpurun_out/full_$k
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $rep \
    python tools/sort_once.py > gpurun_out/ncu_full_$k.log 2>&1
  python tools/ncu_summary.py $rep.ncu-rep gpurun_out/full_$k.md > /dev/null 2>&1
  ncu -i $rep.ncu-rep --page source --csv --print-source=cuda,sass > /tmp/src_$k.csv 2>/dev/null
  python tools/ncu_by_line.py /tmp/src_$k.csv 40 > gpurun_out/full_${k}_lines.txt 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/full_${k}_raw.csv 2>/dev/null
  [ "${KEEP:-0}" = 1 ] || rm -f $rep.ncu-rep
done
echo done
