# ncu launch list + one full capture of the PC kernel + phase/perf probes (diagnostics)
set -x
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pc -s 3 -c 1 \
  -o gpurun_out/prof_ws python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_bench.log 2>&1
timeout 300 python tools/probe_perf.py > gpurun_out/perf.log 2>&1
timeout 300 python tools/probe_phases.py 1000 > gpurun_out/phases.log 2>&1
timeout 300 python tools/probe_phases.py 100000 >> gpurun_out/phases.log 2>&1
cat gpurun_out/perf.log gpurun_out/phases.log
