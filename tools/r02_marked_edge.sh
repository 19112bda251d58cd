# marked-vertex tile test: variants tests + timing (tools/r02_marked_edge.sh <tag>)
tag=$1
timeout 1500 python -m pytest tests/test_gpu_variants.py -q -x -k "lattice" > gpurun_out/${tag}_tests.txt 2>&1; echo rc=$? >> gpurun_out/${tag}_tests.txt
python tools/time_marked.py > gpurun_out/${tag}_marked.txt 2>&1
python tools/time_trace.py 4096 >> gpurun_out/${tag}_marked.txt 2>&1
