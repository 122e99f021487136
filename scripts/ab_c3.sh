# A/B of environment knobs on the C3 step: each argument is "NAME=VALUE ..." (or "base");
# prints the median step time of 6 steps per setting, two alternating passes.
for pass in 1 2; do
  for cfg in "$@"; do
    if [ "$cfg" = base ]; then envs=""; else envs="$cfg"; fi
    ms=$(env $envs timeout 300 python scripts/c3_steps.py 6 0 2>/dev/null | awk '/^step/{print $3}' | sort -n | awk '{a[NR]=$1} END{print a[int((NR+1)/2)]}')
    echo "pass $pass [$cfg] median step ms: $ms"
  done
done
