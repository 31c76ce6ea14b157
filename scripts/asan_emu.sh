#!/bin/bash
# Bounds / undefined-behaviour check of the kernel bodies (compute-sanitizer is
# closed on the GPU pool): the emulation build (the same kernel source as plain
# C++) under AddressSanitizer + UBSan, driven by the CPU parity tests.
set -e
cd "$(dirname "$0")/.."
LIB=$(python paper_2506_19370_b200/build.py --asan | tail -1)
export FCSG_EMU_LIB=$LIB
export LD_PRELOAD="$(gcc -print-file-name=libasan.so) $(gcc -print-file-name=libubsan.so)"
export ASAN_OPTIONS=detect_leaks=0:halt_on_error=1:abort_on_error=1
export UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1
python -m pytest tests/test_kernels.py tests/test_geometries.py tests/test_distributed.py tests/test_fallback_classifier.py \
    tests/test_host.py -m "not gpu" -q -x -p no:cacheprovider "$@"
