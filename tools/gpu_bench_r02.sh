# bench contract checks on one B200: default (C4), C2, self-launched 2 ranks (gloo, shared GPU),
# reference arm; GPU tests of the new drop-in pieces
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "acceptance or caller_operators or dropin or gather" 2>&1 | tail -30 > gpurun_out/pytest_new.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --gpus 2 --dist-backend gloo --config c2 --steps 3 > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt
cat gpurun_out/pytest_new.log; tail -c 3000 gpurun_out/bench_default.json; tail -5 gpurun_out/bench_g2.err
