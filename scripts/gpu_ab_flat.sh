# A/B the full-diamond region pass: layered (region_pass) vs layer-free (flat_node_pass)
set -x
for v in layers nodes; do
  TCG_LIBRARY=$PWD/paper_2604_09221_b200/libtcg_$v.so timeout 600 python scripts/measure_configs.py C5 C4 2>&1 | sed "s/^/$v /"
done
TCG_LIBRARY=$PWD/paper_2604_09221_b200/libtcg_nodes.so timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
