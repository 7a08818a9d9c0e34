# GPU tests + race/perf/phase probes (iteration loop)
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python tools/probe_race.py 160 24 100 > gpurun_out/race.log 2>&1
timeout 300 python tools/probe_perf.py > gpurun_out/perf.log 2>&1
timeout 300 python tools/probe_phases.py 1000 > gpurun_out/phases.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/race.log gpurun_out/perf.log gpurun_out/phases.log
