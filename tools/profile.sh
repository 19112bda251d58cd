#!/bin/bash
# Profiling recipe run under gpurun (one GPU).  usage: tools/profile.sh <tag>
# Each ncu run is preceded by the identical command exiting 0 without ncu; the
# full reports stay in /tmp on the box, their raw/source pages come back as CSV.
set -u
tag=${1:-prof}
out=gpurun_out
mkdir -p $out
B="python bench.py --steps 1 --warmup 3 --walk-steps 20 --no-extras --no-cpu"
$B > $out/${tag}_plain_bench.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/${tag}_launches.csv $B > $out/${tag}_ncu_launches.log 2>&1
bash tools/ncu_capture.sh ${tag}_tb lattice_tb 4 -- $B
bash tools/ncu_capture.sh ${tag}_hc hc_stream 6 -- python tools/run_c4.py 22
echo done
