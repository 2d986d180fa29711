#!/bin/bash
# Phase-profiling variant of the library (K1 clock64 marks): paper_2403_13135_b200/_C/prof/
set -e
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()"
C=paper_2403_13135_b200/_C
mkdir -p $C/prof
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Iinclude -Ipaper_2403_13135_b200/csrc -DICE_AL_PROF -c paper_2403_13135_b200/csrc/autolabel.cu -o $C/prof/autolabel.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $C/prof/libicelabel_b200.so $C/prof/autolabel.o $(ls $C/*.o | grep -v autolabel.o)
