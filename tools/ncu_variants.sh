#!/bin/bash
# DRAM bytes / duration of the JACOBI7 do_all sweep under scheduling variants (one launch each)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct
for cfg in "0 0 0" "16 0 0" "8 0 0" "32 0 0" "64 0 0" "1 2 0" "2 2 0" "4 2 0" "16 0 3"; do
  set -- $cfg
  ncu --metrics $M --clock-control none -k regex:sweep_tma -s 3 -c 1 --csv python tools/sweep_probe.py --ops JACOBI7 --impls 0 --reps 1 --zchunks $1 --sched $2 --l2promo $3 2>/dev/null | grep -E '"(gpu__time|dram__bytes|lts__t)' | awk -F'","' -v c="$cfg" '{printf "%s | %s %s %s\n", c, $(NF-2), $(NF-1), $NF}'
done
