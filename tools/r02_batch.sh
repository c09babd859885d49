# Round-2 (session 2) measurement batch: every BASELINE config plus the
# NEXT-row workloads and Table 1's sweep, one JSON line each, into
# gpurun_out/r02final/.  Usage (on the GPU box): bash tools/r02_batch.sh
set -x
O=gpurun_out/r02final
mkdir -p $O
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
$B --config C1 --steps 20 --warmup 5 > $O/C1.json 2>/dev/null
for d in 5 10 20; do $B --config C2 --deg $d > $O/C2deg$d.json 2>/dev/null; done
$B --config C5 > $O/C5.json 2>/dev/null
$B --config C5 --poly contour > $O/C5polycontour.json 2>/dev/null
$B --config C6 > $O/C6.json 2>/dev/null
python bench.py --config C7 --deg 15 --check-every 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/C7.json 2>/dev/null
for d in 1 2 4 8 16 32 64; do
  k=$((64/d))
  for kr in lanczos lanczos2p; do
    if [ $d = 1 ]; then extra="--plain"; else extra="--deg $((d-1)) --precond right"; fi
    $B --config T1 $extra --krylov $kr --check-every $k > $O/t1_d${d}_$kr.json 2>/dev/null
  done
done
ls $O | wc -l
