# what the driver runs at round end, plus the Fig-2 byte-identity check
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; cat gpurun_out/final_bench.json | cut -c1-400
timeout 400 python bench.py --impl reference | cut -c1-200
bash scripts/gpu_fig2.sh
