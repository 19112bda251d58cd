#!/bin/bash
# usage (under gpurun): tools/ncu_capture.sh <tag> <kernel-regex> <skip> -- <command...>
# Runs <command> once without ncu, then one ncu --set full capture of one launch;
# keeps the report in /tmp and exports raw + SASS-source CSV pages into gpurun_out/.
tag=$1; kre=$2; skip=$3; shift 4
mkdir -p gpurun_out
"$@" > gpurun_out/${tag}_plain.log 2>&1 || { echo "plain run failed" >> gpurun_out/${tag}_plain.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 -o /tmp/${tag} "$@" > gpurun_out/${tag}_ncu.log 2>&1
ncu -i /tmp/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_src.csv 2>/dev/null
ls -la /tmp/${tag}.ncu-rep >> gpurun_out/${tag}_ncu.log
