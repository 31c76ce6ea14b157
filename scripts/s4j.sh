for w in 4 5; do
  echo "== FCSG_WCT_WPC=$w"; FCSG_WCT_WPC=$w timeout 300 python scripts/fc_timing.py 2>&1 | tail -1
  FCSG_WCT_WPC=$w timeout 300 python scripts/fc_batch_timing.py 2>&1 | tail -3
done
