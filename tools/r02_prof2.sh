# usage: tools/r02_prof2.sh <tag>: ncu capture of the flow lattice kernel (2048^2, 40 steps)
set -u
tag=$1
bash tools/ncu_capture.sh ${tag}_flow lattice_flow 2 -- python tools/time_lattice.py 2048 40
