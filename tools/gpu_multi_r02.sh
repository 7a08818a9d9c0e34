# multi-device C-ABI + drop-in checks + full GPU suite
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --gpus 2 --launcher native --devices 0,0 --config c2 --steps 3 > gpurun_out/bench_native2.json 2> gpurun_out/bench_native2.err
timeout 600 ./tests/cpp/ref_acceptance > gpurun_out/ref_acceptance.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/ref_acceptance.log; tail -c 1500 gpurun_out/bench_native2.json; tail -5 gpurun_out/bench_native2.err
