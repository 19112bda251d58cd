#!/bin/bash
# Profiling recipe run under gpurun (one GPU).  usage: tools/profile.sh <tag>
# Each ncu run is preceded by the identical command exiting 0 without ncu.
set -u
tag=${1:-prof}
out=gpurun_out
mkdir -p $out
B="python bench.py --steps 1 --warmup 3 --walk-steps 20 --no-extras --no-cpu"
$B > $out/${tag}_plain_bench.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/${tag}_launches.csv $B > $out/${tag}_ncu_launches.log 2>&1
$B > $out/${tag}_plain_bench2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:lattice_tb -s 4 -c 1 \
    -o $out/${tag}_tb $B > $out/${tag}_ncu_tb.log 2>&1
C="python tools/run_c4.py 22"
$C > $out/${tag}_plain_c4.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:hc_pos -s 6 -c 1 \
    -o $out/${tag}_hc $C > $out/${tag}_ncu_hc.log 2>&1
echo done
