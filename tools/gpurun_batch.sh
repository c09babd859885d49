python -c "import __graft_entry__ as g; g.build()"
( time timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf ) > gpurun_out/r2_gpu_suite2.log 2>&1; echo pytest_rc=$?
tail -6 gpurun_out/r2_gpu_suite2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1; echo ncu_smoke_rc=$?
timeout 900 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2_bench_default.json'));print(d['value'],d['e2e']['value'],d['roofline']['frac'],d['cpu_baseline']['value'],d['clocks'])"
