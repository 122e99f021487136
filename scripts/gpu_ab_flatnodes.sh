# A/B: full-diamond region pass (default) vs layer-free flat node pass (-DTCG_FLAT_NODES) on C5/C4
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python scripts/measure_configs.py C5 C4 2>&1 | cut -c1-200
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DTCG_FLAT_NODES -o paper_2604_09221_b200/libtcg.so paper_2604_09221_b200/csrc/tcg.cu
echo "== TCG_FLAT_NODES"
timeout 600 python scripts/measure_configs.py C5 C4 2>&1 | cut -c1-200
