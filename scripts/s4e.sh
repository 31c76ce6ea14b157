# A/B of wpass.cu knob variants (scripts/build_variant.sh): pass timings
mkdir -p gpurun_out
echo "== default"; timeout 300 python scripts/time_passes_raw.py 2>&1 | tail -3
for v in paper_2506_19370_b200/lib/variants/libfcsg_*.so; do
  echo "== $v"; FCSG_LIB=$PWD/$v timeout 300 python scripts/time_passes_raw.py 2>&1 | tail -3
done
