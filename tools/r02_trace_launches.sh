python tools/time_trace.py 4096 > gpurun_out/r02ca_trace.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r02ca_launches.csv python tools/time_trace.py 4096 > /dev/null 2>&1
