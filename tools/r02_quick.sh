# usage: tools/r02_quick.sh <tag>: lattice timing (flow / per-launch) + lattice parity subset
set -u
tag=$1
mkdir -p gpurun_out
{
for nx in 1024 2048 4096; do python tools/time_lattice.py $nx 1000; done
for nx in 2048 4096; do QWB_LATTICE_FLOW=0 python tools/time_lattice.py $nx 1000; done
} > gpurun_out/${tag}_sweep.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "lattice or subnormal or c2_2048 or trace or slab or search" > gpurun_out/${tag}_gputests.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_gputests.txt
