# round-2 final records: GPU suite, sanitizers, ncu of every config's timed launch, launch list,
# bench lines of every config / mode / C5 leg, reference arms, acceptance, fuzz
set -x
R=gpurun_out/final
mkdir -p $R
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $R/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $R/pytest_gpu.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/race_cases.py 2>&1 | tail -2 > $R/racecheck.log
timeout 900 compute-sanitizer --tool memcheck python tools/race_cases.py 2>&1 | tail -2 > $R/memcheck.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $R/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $R/launch_c4.log 2>&1
for c in "c2" "c4" "c2 --mode augmented_parallel" "c3" "c5 --nodes 64" "c5 --nodes 128" "c5 --nodes 200" "c5 --nodes 256" "c5 --nodes 200 --force n_body"; do
  tag=$(echo $c | sed 's/--mode /_/; s/--nodes /_n/; s/ --force n_body/_newton/; s/ //g')
  skip=4; [ "$tag" = "c3" ] && skip=16
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pc -s $skip -c 1 \
    -o /tmp/prof_$tag python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > $R/prof_$tag.log 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > $R/prof_${tag}_raw.csv 2>/dev/null
done
cp /tmp/prof_c4.ncu-rep $R/ 2>/dev/null
for c in "c1" "c2" "c3" "c4" "c2 --mode augmented_parallel" "c2 --mode grouped" "c4 --mode augmented_parallel" \
         "c5 --nodes 64" "c5 --nodes 96" "c5 --nodes 128" "c5 --nodes 160" "c5 --nodes 200" "c5 --nodes 256" \
         "c5 --nodes 64 --force n_body" "c5 --nodes 96 --force n_body" "c5 --nodes 128 --force n_body" \
         "c5 --nodes 160 --force n_body" "c5 --nodes 200 --force n_body" "c5 --nodes 256 --force n_body"; do
  tag=$(echo $c | sed 's/--mode /_/; s/--nodes /_n/; s/ --force n_body/_newton/; s/ //g')
  timeout 600 python bench.py --config $c > $R/bench_$tag.json 2> $R/bench_$tag.err
done
timeout 600 python bench.py --impl reference > $R/bench_ref_c4.json 2> $R/bench_ref_c4.err
timeout 600 python bench.py --impl reference --config c2 > $R/bench_ref_c2.json 2> $R/bench_ref_c2.err
timeout 600 python bench.py --gpus 2 --dist-backend gloo --config c5 --steps 2 > $R/bench_g2_c5.json 2> $R/bench_g2_c5.err
timeout 600 python bench.py --gpus 2 --launcher native --devices 0,0 --config c2 --steps 3 > $R/bench_native2_c2.json 2> $R/bench_native2_c2.err
timeout 600 ./tests/cpp/ref_acceptance > $R/ref_acceptance.log 2>&1
timeout 900 python tools/fuzz_parity.py 400 31 2>&1 | tail -3 > $R/fuzz.log
lscpu > $R/lscpu.txt
du -sh $R
cat $R/pytest_gpu.log $R/racecheck.log $R/memcheck.log $R/fuzz.log; tail -3 $R/ref_acceptance.log
