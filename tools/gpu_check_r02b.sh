# round-2 re-entry check: full GPU suite, default bench (C4), C2, native 2-context and gloo 2-rank flow checks,
# reference acceptance program, reference arm
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 600 ./tests/cpp/ref_acceptance > gpurun_out/ref_acceptance.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --gpus 2 --launcher native --devices 0,0 --config c2 --steps 3 > gpurun_out/bench_native2.json 2> gpurun_out/bench_native2.err
timeout 600 python bench.py --gpus 2 --dist-backend gloo --config c2 --steps 3 > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
lscpu > gpurun_out/lscpu.txt
cat gpurun_out/pytest_gpu.log | tail -5; tail -20 gpurun_out/ref_acceptance.log
for f in bench_default bench_c2 bench_native2 bench_g2 bench_ref; do echo "== $f"; tail -c 2500 gpurun_out/$f.json; tail -3 gpurun_out/$f.err; done
