python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_resident.py tests/test_gpu_variants.py -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r2_idx16b.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2_idx16b.log
for c in "C5" "C6" "C1" "C2 --deg 5" "C2 --deg 20"; do for f in 1 0; do PPF_IDX16=$f timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_i.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_i.json'));print('$c idx16=$f',round(d['value']*1e3,3),'ms m',d['config']['m'], d['layout']['column_index_bits'], {k:round(v,2) for k,v in d['breakdown_ms_per_step'].items()})"; done; done
