# usage: bash tools/exp_variants.sh OUT v1 v2 ... ("main" = the in-tree library)
out=$1; shift
for v in "$@"; do
  if [ $v = main ]; then unset SABA_LIB; else export SABA_LIB=$PWD/paper_2410_14056_b200/_variants/$v/libsaba_cuda.so; fi
  echo "== $v" >> $out
  python tools/aesc_run.py --workload cfg3 --reps 2 2>&1 | grep aesc: >> $out
  python tools/aesc_run.py --workload cfg4 --sources 64 --reps 2 2>&1 | grep aesc: >> $out
  python tools/aesc_run.py --workload cfg5 --sources 512 --reps 2 2>&1 | grep aesc: >> $out
done
