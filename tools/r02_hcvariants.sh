# usage: tools/r02_hcvariants.sh <tag> <variant.so>...: C4 (hypercube(22)) timing per library variant
set -u
tag=$1; shift
mkdir -p gpurun_out
cp paper_2406_08186_b200/_lib/libqwb200.so /tmp/cur.so
for v in /tmp/cur.so "$@"; do
  cp $v paper_2406_08186_b200/_lib/libqwb200.so
  echo "== $v"
  python tools/run_c4.py 22 | tail -1
done > gpurun_out/${tag}_hcvariants.txt 2>&1
cp /tmp/cur.so paper_2406_08186_b200/_lib/libqwb200.so
