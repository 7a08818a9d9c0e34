# full GPU suite + per-phase cycle breakdowns of the slot kernels (1PN N=64/128/200, Newtonian N=200)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
for a in "20000 planets8 64 1 n_body_1pn" "20000 planets8 128 1 n_body_1pn" "20000 planets8 200 1 n_body_1pn" "20000 planets8 200 1 n_body" "20000 planets8 64 1 n_body"; do
  timeout 300 python tools/probe_phases.py $a >> gpurun_out/phases.log 2>&1
done
cat gpurun_out/pytest_gpu.log gpurun_out/phases.log
