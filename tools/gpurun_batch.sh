python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s -p no:cacheprovider -k C7 > gpurun_out/r2_fullsize_c7.log 2>&1; echo full_rc=$?
grep "^\[\|passed\|failed" gpurun_out/r2_fullsize_c7.log | tail
for c in "C4 8" "C3 8" "C5 8" "C4 2"; do timeout 600 python tools/enqueue_probe.py $c 2>&1 | tail -1; done
