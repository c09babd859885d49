# Timing experiment (not a product path): how much would slice-uniform pair codes save?
# Patches the scratch copy on the GPU box so both rows of a lane take row 0's code (results are
# wrong at grid boundaries; only the chain's time is read), times the C4 / C3 chain, and
# restores the source.  Usage on the GPU box: bash tools/experiments/run_uniform_pairs.sh
O=gpurun_out/${OUT:-r02s4_uniform}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build0.log 2>&1
for c in C4 C3; do python tools/spmv_micro.py --config $c --deg 20 --reps 5; done | tee $O/base.txt
patch -p1 < tools/experiments/uniform_pairs.patch
python -c "from paper_2401_06684_b200 import build; build.build(force=True)" > $O/build1.log 2>&1; echo build_rc=$?
for c in C4 C3; do python tools/spmv_micro.py --config $c --deg 20 --reps 5; done | tee $O/uniform.txt
patch -R -p1 < tools/experiments/uniform_pairs.patch
python -c "from paper_2401_06684_b200 import build; build.build(force=True)" > $O/build2.log 2>&1
for c in C4 C3; do python tools/spmv_micro.py --config $c --deg 20 --reps 5; done | tee $O/base2.txt
