# full ncu capture of the bench-size k_pc_ws launch (skip 3 warm-ups + the 1-trajectory launch-count probe)
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pc -s 4 -c 1 \
  -o gpurun_out/prof_ws2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_bench2.log 2>&1
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/racecheck.log 2>&1
tail -5 gpurun_out/racecheck.log
