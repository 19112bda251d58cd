# usage: tools/r02_variants.sh <tag> <variant.so>...: lattice timing per library variant
set -u
tag=$1; shift
mkdir -p gpurun_out
cp paper_2406_08186_b200/_lib/libqwb200.so /tmp/cur.so
for v in /tmp/cur.so "$@"; do
  cp $v paper_2406_08186_b200/_lib/libqwb200.so
  echo "== $v"
  for nx in 2048 4096; do python tools/time_lattice.py $nx 1000; done
  QWB_LATTICE_FLOW=0 python tools/time_lattice.py 4096 1000
done > gpurun_out/${tag}_variants.txt 2>&1
cp /tmp/cur.so paper_2406_08186_b200/_lib/libqwb200.so
