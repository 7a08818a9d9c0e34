# round-2 baseline: GPU tests + per-config ncu captures (C2, C4, C5 1PN N=64/200) + launch list.
# ncu reports are exported to CSV on the box and deleted (gpurun copies back <= 64 MiB).
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/launch_c2.log 2>&1
for c in "c2" "c4" "c5 --nodes 64" "c5 --nodes 200"; do
  tag=$(echo $c | tr -d ' -')
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pc -s 4 -c 1 \
    -o /tmp/prof_$tag python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_$tag.log 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_$tag.ncu-rep --page details --csv > gpurun_out/prof_${tag}_details.csv 2>/dev/null
done
cp /tmp/prof_c2.ncu-rep gpurun_out/ 2>/dev/null
for c in c2 c4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; done
du -sh gpurun_out
cat gpurun_out/pytest_gpu.log gpurun_out/bench_c2.json gpurun_out/bench_c4.json
