#!/bin/bash
# Build a variant of libdomdec_b200.so into build_<name>/ (loaded with DD_LIB_PATH).
#   scripts/build_variant.sh nt256 "-DDD_NT=256 -DDD_CELL_MIN_BLOCKS=2"
set -e
name=$1; shift
flags="$*"
cd "$(dirname "$0")/../paper_2410_08859_b200/csrc"
out=../../build_$name
mkdir -p $out
ARCH="-gencode arch=compute_100a,code=sm_100a"
F="-O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I../../include --expt-relaxed-constexpr"
nvcc $ARCH $F $flags -c cell.cu -o $out/cell.o -Xptxas -v 2> $out/ptxas_cell.log
nvcc $ARCH $F -c grid.cu -o $out/grid.o
nvcc $ARCH $F $flags -c vol.cu -o $out/vol.o -Xptxas -v 2> $out/ptxas_vol.log
nvcc $ARCH -shared -o $out/libdomdec_b200.so $out/cell.o $out/grid.o $out/vol.o
rm -f $out/*.o
grep -A2 "cell_solve_kernelILi0" $out/ptxas_cell.log | grep -E "registers|spill" || true
grep -A2 "cell_solve3" $out/ptxas_vol.log | grep -E "registers|spill" || true
