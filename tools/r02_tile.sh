# Slice-schedule experiment (pair-code SpMV): C4 and C3 deg 20 with the in-order
# launch and each tile shape, then the new bitwise tests.  Usage: bash tools/r02_tile.sh
O=gpurun_out/${OUT:-r02s4_tile}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build_rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "slice_schedule or pair_codes" > $O/tests.log 2>&1; echo pytest_rc=$?
tail -2 $O/tests.log
for t in 0 4x2 8x1 2x4 0 4x2; do
  PPF_SELLP_TILE=$t timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-alt-layout > $O/c4_$t.json 2> $O/c4_$t.err
  python - <<P
import json
d=json.load(open("$O/c4_$t.json")); print("C4 tile $t", round(d["ms_per_step"],2), d["breakdown_ms_per_step"], d["clocks"]["sm_mhz"])
P
done
for t in 0 4x2 8x1 2x4; do
  PPF_SELLP_TILE=$t timeout 600 python bench.py --config C3 --deg 20 --steps 5 --warmup 3 --no-cpu-baseline --no-alt-layout > $O/c3_$t.json 2> $O/c3_$t.err
  python - <<P
import json
d=json.load(open("$O/c3_$t.json")); print("C3 tile $t", round(d["ms_per_step"],2), d["breakdown_ms_per_step"], d["clocks"]["sm_mhz"])
P
done
