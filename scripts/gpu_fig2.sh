# re-run the three Fig-2 exhaustive 2^42 sweeps and compare the reports byte for byte
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/fig2v${TAG:-x}
for n in bowtie8 fig2-middle8 fig2-right8; do
  timeout 2400 python scripts/fig2_full.py $n --shards 16 --out gpurun_out/fig2v${TAG:-x} > gpurun_out/fig2v${TAG:-x}/$n.log 2>&1
  tail -1 gpurun_out/fig2v${TAG:-x}/$n.log | cut -c1-200
  cmp gpurun_out/fig2v${TAG:-x}/$n.jsonl results/fig2/$n.jsonl && echo "$n jsonl identical"
  cmp gpurun_out/fig2v${TAG:-x}/$n.csv results/fig2/$n.csv && echo "$n csv identical"
done
