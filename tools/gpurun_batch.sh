python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_guards.py tests/test_gpu_variants.py -m gpu -q -s -p no:cacheprovider -rf -k "guard or bitwise or polygon or contour" > gpurun_out/r02/guards.log 2>&1; echo pytest_rc=$?
grep "GPU gaps\|passed\|failed\|FAILED" gpurun_out/r02/guards.log | tail -8
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_c4.json 2> gpurun_out/r02/bench_c4.err; echo c4_rc=$?
for c in "C3 --deg 10" "C3 --deg 20" "C3 --deg 40" "C5" "C1" "C2 --deg 5" "C2 --deg 10" "C2 --deg 20" "C6" "C7" "C5 --poly contour"; do
  f=$(echo $c | tr -d ' -' ); timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_$f.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/r02/bench_$f.json'));print('$c',round(d['value']*1e3,3),'ms m',d['config']['m'],{k:round(v,2) for k,v in d['breakdown_ms_per_step'].items()},{k:round(v or 0) for k,v in d['breakdown_gbs'].items()}, 'frac', round(d['roofline']['frac'] or 0,3))"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02/ncu_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-profile > gpurun_out/r02/ncu_launches.log 2>&1; echo ncu_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled --kernel-name 'regex:sell2_kernel' --launch-skip 200 --launch-count 1 -o gpurun_out/r02/sell2_c4 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-profile > gpurun_out/r02/ncu_sell2.log 2>&1; echo ncu2_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled --kernel-name 'regex:cgs_kernel<double, .int.24, .int.3>' --launch-skip 8 --launch-count 1 -o gpurun_out/r02/cgs_updproj_c4 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-profile > gpurun_out/r02/ncu_cgs.log 2>&1; echo ncu3_rc=$?
