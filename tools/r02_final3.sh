# Round-2 session-3 verification batch (current pair-record code): build, smoke,
# the full GPU suite, the default bench line, the C4 launch list and one ncu
# --set full capture of the pair-code SpMV.  Usage on the GPU box: bash tools/r02_final3.sh
O=gpurun_out/${OUT:-r02s3}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo bench_rc=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/gpu_suite.log 2>&1; echo pytest_rc=$?
tail -3 $O/gpu_suite.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
  --log-file $O/launches_c4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-alt-layout --no-profile > $O/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sellp_kernel -s 40 -c 1 \
  -o $O/sellp_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-alt-layout --no-profile > $O/ncu_full.log 2>&1; echo ncu2_rc=$?
