#!/bin/bash
# Sweep walk-kernel variants (profiling helper): hub table size at 1024-thread blocks.
for v in "hthreads=1024,hcount=24576" "hthreads=1024,hcount=32767" "hthreads=1024,hcount=36864" "hthreads=1024,hcount=40960" "hthreads=1024,hcount=45056" "hthreads=1024,hcount=49152" "hthreads=512,hcount=16383"; do
  echo "== cfg2 $v"; SABA_WALK_VARIANT=$v python tools/profile_campaign.py --reps 3 | tail -1
done
