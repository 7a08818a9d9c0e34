# refresh the C5 1PN records (bench lines + ncu of the timed launch) after a k_pc_uni change;
# writes into gpurun_out/final next to the rest of the final records (tools/collect_records.py)
set -x
R=gpurun_out/final
mkdir -p $R
for c in "c5 --nodes 64" "c5 --nodes 128" "c5 --nodes 200" "c5 --nodes 256"; do
  tag=$(echo $c | sed 's/--nodes /_n/; s/ //g')
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pc -s 4 -c 1 \
    -o /tmp/prof_$tag python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > $R/prof_$tag.log 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > $R/prof_${tag}_raw.csv 2>/dev/null
done
for n in 64 96 128 160 200 256; do
  timeout 600 python bench.py --config c5 --nodes $n > $R/bench_c5_n$n.json 2> $R/bench_c5_n$n.err
done
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $R/pytest_gpu.log
cat $R/pytest_gpu.log
