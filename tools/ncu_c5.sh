#!/usr/bin/env bash
# ncu captures of the C5 batch (32 tiles, one eager ILT iteration) on the GPU
# box: launch list + `--set full` of the named kernels, exported as CSV into
# gpurun_out/ for tools/ncu_summarize.py.   usage: tools/ncu_c5.sh [kernel ...]
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out
mkdir -p $OUT
CFG=${CFG:-c5}
TILES=${TILES:-32}
KS=${*:-resist_rows adj_rows socs_rows grad_rows}
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $OUT/launches.csv python tools/prof_c5.py --config $CFG --tiles $TILES > $OUT/ncu_launch.log 2>&1
for k in $KS; do
  ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:fk_${k} -c 1 \
      -f -o $OUT/cap_$k python tools/prof_c5.py --config $CFG --tiles $TILES > $OUT/ncu_$k.log 2>&1
  ncu -i $OUT/cap_$k.ncu-rep --page raw --csv > $OUT/raw_$k.csv 2>/dev/null
  ncu -i $OUT/cap_$k.ncu-rep --page details --csv > $OUT/details_$k.csv 2>/dev/null
  ncu -i $OUT/cap_$k.ncu-rep --page source --csv > $OUT/source_$k.csv 2>/dev/null
  mkdir -p /tmp/ncu_reps && mv $OUT/cap_$k.ncu-rep /tmp/ncu_reps/  # reps stay on the box (size cap)
done
ls -la $OUT
