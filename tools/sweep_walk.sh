#!/bin/bash
# Sweep walk-kernel variants (profiling helper).
for v in "wpt=4,packed=1,agg=1" "wpt=2,packed=1,agg=1" "wpt=4,packed=1,agg=0"; do
  echo "== cfg2 $v"; SABA_WALK_VARIANT=$v python tools/profile_campaign.py --reps 3 | tail -1
done
echo "== cfg1 auto"; python tools/profile_campaign.py --reps 3 --workload cfg1 | tail -1
