# A/B of library builds on the C3 step: each argument is a build/ library name
for pass in 1 2; do
  for lib in "$@"; do
    ms=$(TCG_LIBRARY=build/$lib timeout 300 python scripts/c3_steps.py 5 1 2>/dev/null | awk '/^step/{print $3, $12}' | sort -n | sed -n 3p)
    echo "pass $pass [$lib] median step ms / l15: $ms"
  done
done
