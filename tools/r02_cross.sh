# usage: tools/r02_cross.sh <tag>: flow vs per-launch lattice timing over sizes, then the GPU suite
set -u
tag=$1
mkdir -p gpurun_out
{
for nx in 512 768 1024 1536 2048 3072 4096; do
  python tools/time_lattice.py $nx 1000
  QWB_LATTICE_FLOW=0 python tools/time_lattice.py $nx 1000
done
} > gpurun_out/${tag}_cross.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_gputests.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_gputests.txt
