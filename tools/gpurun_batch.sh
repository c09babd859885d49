python -c "import __graft_entry__ as g; g.build()"
timeout 1700 python -m pytest tests/test_gpu_peer.py tests/test_gpu_multirank.py tests/test_gpu_bench_dist.py tests/test_gpu_sharded.py tests/test_gpu_guards.py -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2_peer.log 2>&1; echo pytest_rc=$?
tail -8 gpurun_out/r2_peer.log
