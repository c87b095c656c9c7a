# A/B of the count variants (scripts/count_variants.py) under environment knobs.
mkdir -p gpurun_out
for cfg in ${CFGS:-c5 c2}; do
  python scripts/count_variants.py $cfg
  SEL_PREFETCH=1 python scripts/count_variants.py $cfg
  SEL_PREFETCH=0 python scripts/count_variants.py $cfg
  SEL_FAST=0 python scripts/count_variants.py $cfg
  SEL_CTAS_PER_SM=3 python scripts/count_variants.py $cfg
  SEL_CTAS_PER_SM=2 python scripts/count_variants.py $cfg
done
