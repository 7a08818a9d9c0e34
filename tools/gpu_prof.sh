# ncu launch list of the bench command + one full capture of the bench-size PC launch
# (skip the 3 warm-ups and the 1-trajectory launch-count probe) + GPU tests
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pc -s 4 -c 1 \
  -o gpurun_out/prof_ws python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_bench.log 2>&1
cat gpurun_out/pytest_gpu.log
