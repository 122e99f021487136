# dump the SASS of one kernel: scripts/sass_fn.sh <lib.so> <name-regex>
cuobjdump -sass "$1" | awk -v pat="$2" '/Function :/ {p = ($0 ~ pat)} p'
