#!/bin/bash
# usage: tools/ptxas_check.sh <file.cu> [grep-pattern]  — registers/spills per kernel
f=$1; pat=${2:-.}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC \
  -Xptxas -v -c "$f" -o /tmp/ptxas_check.o 2>&1 | grep -E "error|registers|spill|Compiling" | paste - - - \
  | grep -E "$pat" | sed -E 's/.*entry function .(_Z[^ ]*). for.*stack frame, ([0-9]+) bytes spill stores.*Used ([0-9]+) registers.*/\1 spill=\2 regs=\3/'
