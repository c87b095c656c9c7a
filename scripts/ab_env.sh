# bench.py step times under library variants x environment settings.
# Usage: scripts/ab_env.sh "c2 c5" "base st2" "X=1 Y=0" ...    (base = in-tree libsel.so; "-" = no env)
CFGS=$1; LIBS=$2; shift 2
for cfg in $CFGS; do
  for v in $LIBS; do
    for e in "$@"; do
      lib=""; [ "$v" != base ] && lib="SEL_LIB=$PWD/build_exp/libsel_$v.so"
      envs=""; [ "$e" != "-" ] && envs="$e"
      env $lib $envs timeout 300 python bench.py --steps 20 --warmup 5 --config $cfg --no-e2e --no-cpu --no-read-peak 2>&1 | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $v [$e]', d['ms_per_step'], d['latency_ms']['count_kernel'], d['latency_ms']['pushdown_kernels'])" 2>&1 | tail -1
    done
  done
done
