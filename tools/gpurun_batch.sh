python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r02
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02/ncu_launches_c4_idx16.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-profile > /dev/null 2>&1; echo ncu_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled --kernel-name 'regex:sell2_kernel' --launch-skip 200 --launch-count 1 -o gpurun_out/r02/sell2_c4_idx16 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-profile > /dev/null 2>&1; echo ncu2_rc=$?
