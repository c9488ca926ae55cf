#!/bin/bash
# Sweep campaign kernel variants on cfg2 (profiling helper): walk_kernel_ms per rep.
# usage: tools/sweep_walk.sh "variant1" "variant2" ...   ("" = default)
for v in "$@"; do
  echo "== cfg2 [$v]"; SABA_WALK_VARIANT=$v python tools/profile_campaign.py --reps 4 | tail -2
done
