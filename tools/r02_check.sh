# usage: tools/r02_check.sh <tag> [pytest-args...]: GPU tests + lattice sweep
set -u
tag=$1; shift
mkdir -p gpurun_out
for nx in 1024 2048 4096; do python tools/time_lattice.py $nx 1000; done > gpurun_out/${tag}_sweep.txt 2>&1
QWB_LATTICE_FLOW=0 python tools/time_lattice.py 2048 1000 >> gpurun_out/${tag}_sweep.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x "$@" > gpurun_out/${tag}_gputests.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_gputests.txt
