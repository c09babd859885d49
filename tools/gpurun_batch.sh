python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_multirank.py tests/test_gpu_peer.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_pytest4.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2_pytest4.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench4.json 2> gpurun_out/r2_bench4.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2_bench4.json'));print(d['value'],d['breakdown_ms_per_step'],d['breakdown_gbs'])"
for c in "C2 --deg 5" "C7"; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench4_x.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_bench4_x.json'));print('$c',d['value'],d['config']['m'],d['breakdown_ms_per_step'],d['breakdown_gbs'])"; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled --kernel-name 'regex:cgs_kernel' --csv --log-file gpurun_out/r2_cgs_launches4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-profile > gpurun_out/r2_ncu_cgs5.log 2>&1; echo ncu_rc=$?
