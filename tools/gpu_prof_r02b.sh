# ncu --set full of the TIMED step's solve launch of each config (warm-up launches 0..W-1, the
# 1-trajectory launch-count probe next, then the timed step), exported to CSV on the box
set -x
mkdir -p gpurun_out/rec
for c in "c2" "c4" "c2 --mode augmented_parallel" "c5 --nodes 64" "c5 --nodes 128" "c5 --nodes 200" "c5 --nodes 256" "c3"; do
  tag=$(echo $c | sed 's/--mode /_/; s/--nodes /_n/; s/ //g')
  skip=4; [ "$tag" = "c3" ] && skip=16
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pc -s $skip -c 1 \
    -o /tmp/prof_$tag python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/rec/prof_$tag.log 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/rec/prof_${tag}_raw.csv 2>/dev/null
done
cp /tmp/prof_c4.ncu-rep gpurun_out/rec/ 2>/dev/null
timeout 600 python bench.py --config c5 --nodes 256 > gpurun_out/rec/bench_c5_n256.json 2> gpurun_out/rec/bench_c5_n256.err
du -sh gpurun_out/rec
