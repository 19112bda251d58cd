# flow kernel: per-step time vs run length, with SM clocks sampled
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 100 > gpurun_out/r02ab_smi.csv &
SMI=$!
for st in 40 200 1000; do
  echo "steps $st"; QWB_LATTICE_FLOW=2 python tools/time_lattice.py 4096 $st; QWB_LATTICE_FLOW=0 python tools/time_lattice.py 4096 $st
  date +%s.%N
done > gpurun_out/r02ab_flowlen.txt 2>&1
kill $SMI
