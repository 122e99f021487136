# A/B: chunk index limit (TCG_CHUNK_INDEX_LOG2) with the matching bench slice
python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out
for cfg in "33 4" "34 2"; do set -- $cfg
  TCG_CHUNK_INDEX_LOG2=$1 timeout 600 python bench.py --slice-log2 $1 --steps $2 --warmup 3 --no-cpu-baseline > gpurun_out/abc.json 2> gpurun_out/abc.err
  echo "chunk/slice 2^$1 x $2"; grep -E "kernel ms by kind" gpurun_out/abc.err | tail -1; tail -2 gpurun_out/abc.err | cut -c1-300
  python -c "import json; d=json.load(open('gpurun_out/abc.json')); print('  value %.4g e2e %.4g' % (d['value'], d['e2e']['value']), d['parity'], d['roofline']['dedup']['factor'])"
done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
