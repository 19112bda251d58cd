# usage: tools/r02_prof3.sh <tag> <nx>: ncu --set full of the flow kernel and one per-launch kernel
set -u
tag=$1; nx=$2
bash tools/ncu_capture.sh ${tag}_flow lattice_flow 2 -- python tools/time_lattice.py $nx 40
QWB_LATTICE_FLOW=0 bash tools/ncu_capture.sh ${tag}_tb lattice_tb 8 -- python tools/time_lattice.py $nx 40
