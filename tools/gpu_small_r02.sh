# records after the two-CTA small-N variants: C5 N = 64 / 96 / 128 both force models + ncu of N = 64
set -x
R=gpurun_out/small
mkdir -p $R
for c in "c5 --nodes 64" "c5 --nodes 96" "c5 --nodes 128" "c5 --nodes 64 --force n_body" "c5 --nodes 96 --force n_body" "c5 --nodes 128 --force n_body"; do
  tag=$(echo $c | sed 's/--nodes /_n/; s/ --force n_body/_newton/; s/ //g')
  timeout 600 python bench.py --config $c > $R/bench_$tag.json 2> $R/bench_$tag.err
done
for c in "c5 --nodes 64" "c5 --nodes 64 --force n_body"; do
  tag=$(echo $c | sed 's/--nodes /_n/; s/ --force n_body/_newton/; s/ //g')
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pc -s 4 -c 1 \
    -o /tmp/prof_$tag python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > $R/prof_$tag.log 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > $R/prof_${tag}_raw.csv 2>/dev/null
done
