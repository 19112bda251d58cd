# usage: tools/r02_prof.sh <tag>: ncu captures of the per-launch (FLOW=0) and flow lattice kernels, new and old lib
set -u
tag=$1
export QWB_LATTICE_FLOW=0
bash tools/ncu_capture.sh ${tag}_tb lattice_tb 8 -- python tools/time_lattice.py 2048 40
unset QWB_LATTICE_FLOW
bash tools/ncu_capture.sh ${tag}_flow lattice_flow 2 -- python tools/time_lattice.py 2048 40
cp paper_2406_08186_b200/_lib/libqwb200.so /tmp/cur.so
cp exp_libs/old.so paper_2406_08186_b200/_lib/libqwb200.so
bash tools/ncu_capture.sh ${tag}_old lattice_tb 8 -- python tools/time_lattice.py 2048 40
cp /tmp/cur.so paper_2406_08186_b200/_lib/libqwb200.so
