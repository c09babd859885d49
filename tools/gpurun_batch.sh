python -c "import __graft_entry__ as g; g.build()"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c1_launches.csv python bench.py --config C1 --steps 2 --warmup 3 --no-cpu-baseline --no-profile > gpurun_out/r2_c1_ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/r2_c1_ncu.log
timeout 300 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_c1.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/r2_c1.json'));print('C1',round(d['value']*1e3,4),'ms m',d['config']['m'])"
timeout 600 python -m pytest tests/test_gpu_resident.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
