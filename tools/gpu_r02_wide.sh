# wide groups on the slot kernels (member-level rounds) + independent error order: GPU tests,
# reference acceptance program, bench C2/C4 in the grouped / augmented modes
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "wide or group or augmented or error_order or nonconvergence or divergence or singular or timeout" 2>&1 | tail -30 > gpurun_out/pytest_wide.log
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 600 ./tests/cpp/ref_acceptance > gpurun_out/ref_acceptance.log 2>&1
for m in independent augmented_parallel grouped; do
  timeout 300 python bench.py --config c2 --mode $m --no-cpu-baseline > gpurun_out/bench_c2_$m.json 2> gpurun_out/bench_c2_$m.err
done
timeout 600 python bench.py --config c4 --mode augmented_parallel --no-cpu-baseline --steps 3 > gpurun_out/bench_c4_aug.json 2> gpurun_out/bench_c4_aug.err
cat gpurun_out/pytest_wide.log gpurun_out/pytest_gpu.log | tail -40; tail -12 gpurun_out/ref_acceptance.log
for f in bench_c2_independent bench_c2_augmented_parallel bench_c2_grouped bench_c4_aug; do echo "== $f"; python -c "
import json,sys
d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['kernel'], d.get('parity'), d['config'].get('mode'))
" ; tail -3 gpurun_out/$f.err; done
