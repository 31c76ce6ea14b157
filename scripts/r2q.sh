for rep in 1 2; do
for v in best xkl2 ykc2 ykc8; do
  echo "== $v"; FCSG_LIB=paper_2506_19370_b200/lib/ab_$v.so timeout 600 python scripts/time_groups.py 2>&1 | grep -E "config5|pass_"
done; done
