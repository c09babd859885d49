# Round-2 session-4 closing batch (HEAD with the optional slice schedule): build, smoke,
# the default bench line, the full GPU suite.  Usage on the GPU box: bash tools/r02_final4.sh
O=gpurun_out/${OUT:-r02s4b}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo bench_rc=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/gpu_suite.log 2>&1; echo pytest_rc=$?
tail -3 $O/gpu_suite.log
