#!/bin/bash
# Sweep walk-kernel variants (profiling helper).
for v in "hot=0" "hot=1" "hot=1,agg=0" "hot=1,packed=0"; do
  echo "== cfg2 $v"; SABA_WALK_VARIANT=$v python tools/profile_campaign.py --reps 3 | tail -1
done
echo "== cfg1 fat=0,hot=1"; SABA_WALK_VARIANT=fat=0,hot=1 python tools/profile_campaign.py --reps 3 --workload cfg1 | tail -1
