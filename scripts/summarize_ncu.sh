#!/bin/bash
# Summarize an ncu report into a text file: headline metrics, stall reasons, hottest SASS, regions, DRAM bytes.
# Usage: scripts/summarize_ncu.sh REP.ncu-rep "title line" > out.txt
REP=$1; TITLE=$2
echo "# $TITLE"
python scripts/sass_hot.py "$REP" 25
echo
echo "# instruction regions (scripts/ncu_regions.py)"
python scripts/ncu_regions.py "$REP" 0.7
echo
echo "# raw"
ncu -i "$REP" --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2] if len(r)>2 else r[1]
for k in ['dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__thread_inst_executed_per_inst_executed.ratio','l1tex__t_sector_hit_rate.pct','lts__t_sector_hit_rate.pct','l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','sm__cycles_elapsed.avg.per_second','sm__inst_executed.sum']:
  if k in h: i=h.index(k); print(k, v[i], r[1][i])
"
