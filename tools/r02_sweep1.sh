set -u
mkdir -p gpurun_out
(free -g; nproc; lscpu | head -20; nvidia-smi -L) > gpurun_out/r02a_host.txt 2>&1
for nx in 1024 1536 2048 3072 4096; do python tools/time_lattice.py $nx 240; done > gpurun_out/r02a_sweep.txt 2>&1
QWB_LATTICE_T=0 python tools/time_lattice.py 2048 240 >> gpurun_out/r02a_sweep.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_gputests.txt 2>&1
echo rc=$?
