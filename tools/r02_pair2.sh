# Paired-chain SpMV (sellp_pair_kernel) check and measurement on the GPU box:
# build, the bitwise/oracle tests, then C4 and C3 deg 20 with and without
# pairing and a few handout slacks.  Usage: bash tools/r02_pair2.sh
O=gpurun_out/r02p2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build_rc=$?
timeout 600 python -m pytest tests/test_gpu_pair2.py -m gpu -q -p no:cacheprovider -rf -x -s > $O/tests.log 2>&1; echo pytest_rc=$?
tail -5 $O/tests.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-alt-layout"
for cfg in "C4" "C3 --deg 20"; do
  for v in "PPF_PAIR2=0" "PPF_PAIR2=1" "PPF_PAIR2=1 PPF_PAIR2_SLACK=64" "PPF_PAIR2=1 PPF_PAIR2_SLACK=1500"; do
    tag=$(echo "$cfg $v" | tr ' =' '__')
    env $v timeout 300 $B --config $cfg > $O/$tag.json 2> $O/$tag.err
    python -c "import json;d=json.loads(open('$O/$tag.json').read().strip().splitlines()[-1]);print('$cfg $v', round(d['value']*1e3,2),'ms m',d['config']['m'],{k:round(v,2) for k,v in d['breakdown_ms_per_step'].items()}, 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 $O/$tag.err
  done
done
