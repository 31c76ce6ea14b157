#!/bin/bash
# A/B variant of libfcsg.so with different -D knobs for wpass.cu:
#   bash scripts/build_variant.sh NAME -DFCSG_X_MINB=4 -DFCSG_X_KC=2 ...
# -> paper_2506_19370_b200/lib/variants/libfcsg_NAME.so (run with FCSG_LIB=that path)
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p paper_2506_19370_b200/lib/variants build/variants
C=paper_2506_19370_b200/csrc
nvcc -gencode=arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xptxas=-v -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I$C -Iinclude "$@" -c $C/wpass.cu -o build/variants/wpass_$name.o 2>&1 | grep -A1 "wpass_[xy]_kernel" | grep "Used\|spill" | sed 's/ptxas info    ://'
objs=$(ls build/obj/*.o | grep -v "/wpass.cu.o")
nvcc -gencode=arch=compute_100a,code=sm_100a -shared -o paper_2506_19370_b200/lib/variants/libfcsg_$name.so $objs build/variants/wpass_$name.o -lquadmath -ldl -cudart static
echo built $name
