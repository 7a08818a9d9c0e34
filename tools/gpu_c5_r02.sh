# C5 records: 1PN and Newtonian node sweeps, ncu of the Newtonian N = 200 and 1PN N = 64 / 256 launches,
# 2-rank interleaved-shard flow check (gloo, ranks sharing the GPU)
set -x
mkdir -p gpurun_out/c5
for n in 64 96 128 160 200 256; do
  timeout 600 python bench.py --config c5 --nodes $n > gpurun_out/c5/bench_c5_n$n.json 2> gpurun_out/c5/bench_c5_n$n.err
  timeout 600 python bench.py --config c5 --nodes $n --force n_body > gpurun_out/c5/bench_c5_n${n}_newton.json 2> gpurun_out/c5/bench_c5_n${n}_newton.err
done
for c in "--nodes 64" "--nodes 256" "--nodes 200 --force n_body"; do
  tag=$(echo $c | sed 's/--nodes /n/; s/ --force n_body/_newton/')
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pc -s 4 -c 1 \
    -o /tmp/prof_c5_$tag python bench.py --config c5 $c --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c5/prof_c5_$tag.log 2>&1
  ncu -i /tmp/prof_c5_$tag.ncu-rep --page raw --csv > gpurun_out/c5/prof_c5_${tag}_raw.csv 2>/dev/null
done
timeout 600 python bench.py --gpus 2 --dist-backend gloo --config c5 --steps 2 > gpurun_out/c5/bench_g2_c5.json 2> gpurun_out/c5/bench_g2_c5.err
for f in gpurun_out/c5/bench_*.json; do echo "$f $(tail -c 300 $f | head -c 120)"; done
