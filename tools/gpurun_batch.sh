python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py tests/test_gpu_resident.py -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2_wide2.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/r2_wide2.log
timeout 600 python bench.py --config C7 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_C7_wide.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r02_bench_C7_wide.json'));print('C7',round(d['value']*1e3,3),'ms m',d['config']['m'],{k:round(v,2) for k,v in d['breakdown_ms_per_step'].items()},{k:round(v or 0) for k,v in d['breakdown_gbs'].items()})"
