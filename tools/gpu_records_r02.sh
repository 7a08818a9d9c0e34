# round-2 records: GPU suite, per-config ncu captures (exported to CSV on the box), the launch
# list of the default bench, bench lines of every config / mode, reference arm, C3 parity probe
set -x
mkdir -p gpurun_out/rec
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/rec/gpu.txt
lscpu > gpurun_out/rec/lscpu.txt
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/rec/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/rec/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/rec/launch_c4.log 2>&1
for c in "c2" "c4" "c2 --mode augmented_parallel" "c5 --nodes 64" "c5 --nodes 128" "c5 --nodes 200" "c3"; do
  tag=$(echo $c | sed 's/--mode /_/; s/--nodes /_n/; s/ //g')
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pc -s 3 -c 1 \
    -o /tmp/prof_$tag python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/rec/prof_$tag.log 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/rec/prof_${tag}_raw.csv 2>/dev/null
done
cp /tmp/prof_c4.ncu-rep gpurun_out/rec/ 2>/dev/null
for c in "c1" "c2" "c3" "c4" "c2 --mode augmented_parallel" "c2 --mode grouped" "c4 --mode augmented_parallel" \
         "c5 --nodes 64" "c5 --nodes 96" "c5 --nodes 128" "c5 --nodes 160" "c5 --nodes 200" "c5 --nodes 256"; do
  tag=$(echo $c | sed 's/--mode /_/; s/--nodes /_n/; s/ //g')
  timeout 600 python bench.py --config $c > gpurun_out/rec/bench_$tag.json 2> gpurun_out/rec/bench_$tag.err
done
timeout 600 python bench.py --impl reference > gpurun_out/rec/bench_ref_c4.json 2> gpurun_out/rec/bench_ref_c4.err
timeout 600 python bench.py --impl reference --config c2 > gpurun_out/rec/bench_ref_c2.json 2> gpurun_out/rec/bench_ref_c2.err
timeout 900 python tools/probe_c3_parity.py 1000 > gpurun_out/rec/c3_parity.json 2> gpurun_out/rec/c3_parity.err
timeout 600 ./tests/cpp/ref_acceptance > gpurun_out/rec/ref_acceptance.log 2>&1
du -sh gpurun_out/rec
cat gpurun_out/rec/pytest_gpu.log
for f in gpurun_out/rec/bench_*.json; do echo "$f $(tail -c 400 $f | head -c 200)"; done
