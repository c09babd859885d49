# Look-ahead distance of the pair-code SpMV's L2 prefetches (PPF_SELLP_AHEAD, slices; 0 = own slice)
O=gpurun_out/${OUT:-r02s4_ahead}
mkdir -p $O
patch -p1 < tools/experiments/prefetch_ahead.patch   # (scratch copy on the GPU box only)
python -c "from paper_2401_06684_b200 import build; build.build(force=True)" > $O/build.log 2>&1
for a in 0 1184 2368 4736 9472 14208 18944 0; do
  for c in C4 C3; do echo -n "ahead $a: "; PPF_SELLP_AHEAD=$a python tools/spmv_micro.py --config $c --deg 20 --reps 5; done
done | tee $O/ahead.txt
