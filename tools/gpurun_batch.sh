python -c "import __graft_entry__ as g; g.build()"
( time timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf ) > gpurun_out/r2_gpu_suite3.log 2>&1; echo pytest_rc=$?
tail -6 gpurun_out/r2_gpu_suite3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
