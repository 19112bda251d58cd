# usage: tools/sweep_lattice.sh "shape T" ...   (kernel variant sweep: device time per coined step)
for cfg in "$@"; do
  set -- $cfg
  if [ "$1" = "wf" ]; then export QWB_LATTICE_KIND=wf; unset QWB_LATTICE_SHAPE; else unset QWB_LATTICE_KIND; export QWB_LATTICE_SHAPE=$1; fi
  export QWB_LATTICE_T=$2
  for nx in 2048 4096; do
    echo "shape $1 T $2: $(timeout 120 python tools/time_lattice.py $nx 2>&1 | tail -1)" >> gpurun_out/sweep.log
  done
done
