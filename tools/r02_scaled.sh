# Pre-scaled pair codes (ppf_mat::code_scaled): parity tests, then C4 / C3 deg 20
# with PPF_SELLP_SCALED=0/1 alternated.  Usage on the GPU box: bash tools/r02_scaled.sh
O=gpurun_out/r02sc
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build_rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rf -x -k "pair_codes or chebyshev_chain or run_parity_true" > $O/tests.log 2>&1; echo pytest_rc=$?
tail -3 $O/tests.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-alt-layout --no-profile"
for rep in 1 2; do
for cfg in "C4" "C3 --deg 20"; do
  for v in "PPF_SELLP_SCALED=0" "PPF_SELLP_SCALED=1"; do
    tag=$(echo "$cfg $v $rep" | tr ' =' '__')
    env $v timeout 300 $B --config $cfg > $O/$tag.json 2> $O/$tag.err
    python -c "import json;d=json.loads(open('$O/$tag.json').read().strip().splitlines()[-1]);print('$cfg $v', round(d['value']*1e3,2),'ms m',d['config']['m'], d['clocks']['sm_mhz'])" || tail -3 $O/$tag.err
  done
done
done
