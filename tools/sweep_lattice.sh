# usage: tools/sweep_lattice.sh "shape T" ...   (kernel variant sweep, 2048^2 flip-flop)
for cfg in "$@"; do
  set -- $cfg
  if [ "$1" = "wf" ]; then export QWB_LATTICE_KIND=wf; unset QWB_LATTICE_SHAPE; else unset QWB_LATTICE_KIND; export QWB_LATTICE_SHAPE=$1; fi
  export QWB_LATTICE_T=$2
  v=$(timeout 120 python bench.py --steps 5 --warmup 3 --walk-steps 240 --no-extras --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value']/1e9,1), round(d['roofline']['time_per_launch_us'],1))")
  echo "$cfg -> $v" >> gpurun_out/sweep.log
done
