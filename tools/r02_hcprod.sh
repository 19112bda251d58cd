# hc_stream producer-warp variants: parity tests + timing (tools/r02_hcprod.sh <tag>)
set -u
tag=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "hypercube or c4" > gpurun_out/${tag}_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/${tag}_tests.txt
for v in ${VARIANTS:-52 42 51 21202}; do
  echo "== $v"; QWB_HC_STREAM=$v timeout 300 python tools/run_c4.py 22 | tail -2
done > gpurun_out/${tag}_hcprod.txt 2>&1
