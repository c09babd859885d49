set -x
mkdir -p gpurun_out/final
B="python bench.py --steps 5 --warmup 3"
$B --config C1 --steps 20 --warmup 5 > gpurun_out/final/r01_bench_c1.json 2>/dev/null
for d in 5 10 20; do $B --config C2 --deg $d --no-cpu-baseline > gpurun_out/final/r01_bench_c2_deg$d.json 2>/dev/null; done
for d in 10 20 40; do x=""; [ $d != 20 ] && x="--no-cpu-baseline"; $B --config C3 --deg $d $x > gpurun_out/final/r01_bench_c3_deg$d.json 2>/dev/null; done
$B --config C5 > gpurun_out/final/r01_bench_c5.json 2>/dev/null
python bench.py --config C7 --deg 15 --check-every 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final/r01_bench_c7_graph.json 2>/dev/null
for d in 1 2 4 8 16 32 64; do
  k=$((64/d))
  for kr in lanczos lanczos2p; do
    if [ $d = 1 ]; then extra="--plain"; else extra="--deg $((d-1)) --precond right"; fi
    $B --config T1 $extra --krylov $kr --check-every $k --no-cpu-baseline > gpurun_out/final/t1_d${d}_$kr.json 2>/dev/null
  done
done
ls gpurun_out/final | wc -l
