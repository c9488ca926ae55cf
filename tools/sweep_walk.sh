#!/bin/bash
# Sweep walk-kernel variants on cfg2 (profiling helper).
for v in "wpt=4,packed=0,c32=0,agg=1" "wpt=4,packed=1,c32=0,agg=1" "wpt=4,packed=1,c32=1,agg=1" \
         "wpt=4,packed=1,c32=1,agg=0" "wpt=2,packed=1,c32=1,agg=0" "wpt=8,packed=1,c32=1,agg=0" \
         "wpt=1,packed=1,c32=1,agg=0" "wpt=2,packed=1,c32=1,agg=1" "wpt=8,packed=1,c32=1,agg=1"; do
  echo "== $v"; SABA_WALK_VARIANT=$v python tools/profile_campaign.py --reps 3 | tail -1
done
echo "== fetch32"; SABA_L2_FETCH=32 python tools/profile_campaign.py --reps 3 | tail -1
echo "== hash mode"; python tools/profile_campaign.py --reps 3 --mode hash | tail -1
echo "== cfg1"; python tools/profile_campaign.py --reps 3 --workload cfg1 | tail -1
