# count_variants.py under library variants: scripts/ab_count_libs.sh "c5 c2" base noT ...
CFGS=$1; shift
for cfg in $CFGS; do
  for v in "$@"; do
    lib=""; [ "$v" != base ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
    echo -n "$v "; env $lib timeout 300 python scripts/count_variants.py $cfg 2>&1 | tail -1
  done
done
