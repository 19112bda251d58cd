# Build exp_libs/tl.so here (not on the GPU box: build/ does not travel): the
# library with lattice_tb.cu compiled -DQWB_EXP_TIMING (cycle counters and the
# launch timeline, tools/r02_flowdbg.py / tools/r02_timeline.py).  Run after
# `python -c "from paper_2406_08186_b200 import _build; _build.build()"`.
set -e
mkdir -p exp_libs
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC,-O2 -I include \
  -DQWB_EXP_TIMING -c paper_2406_08186_b200/csrc/lattice_tb.cu -o /tmp/ltb_tl.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o exp_libs/tl.so \
  $(ls build/obj/*.o | grep -v lattice_tb) /tmp/ltb_tl.o
