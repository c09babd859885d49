python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "flat or tiny" > gpurun_out/r2_pytest8.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/r2_pytest8.log
for c in "C2 --deg 5" "C2 --deg 10"; do for f in 1 0; do PPF_CGS_FLAT=$f timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-profile > gpurun_out/r2_bench5_x.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_bench5_x.json'));print('$c flat=$f',round(d['value']*1e3,3),'ms m',d['config']['m'])"; done; done
PPF_CGS_FLAT=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c2d5_flat1c.csv python bench.py --config C2 --deg 5 --steps 1 --warmup 3 --no-cpu-baseline --no-profile > /dev/null 2>&1; echo ncu_rc=$?
