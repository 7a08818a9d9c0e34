# Every BASELINE config on one B200 (records for profiles/); N-sweep for C5.
set -x
timeout 600 python bench.py --config c2 --steps 100 --warmup 10 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config c1 --steps 50 --warmup 5 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 900 python bench.py --config c3 --steps 3 --warmup 1 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --config c4 --steps 3 --warmup 1 --cpu-sample 1000 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
for n in 64 96 128 160 200 256; do
  timeout 900 python bench.py --config c5 --nodes $n --steps 3 --warmup 1 --cpu-sample 400 > gpurun_out/bench_c5_n$n.json 2> gpurun_out/bench_c5_n$n.err
done
timeout 600 python bench.py --impl reference --config c2 --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2>&1
tail -c 400 gpurun_out/*.err
for f in gpurun_out/bench_c*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d['roofline']; c=d['cpu_baseline'] or {}
print('$f', d['value'], 'e2e', d['e2e']['value'], 'frac', r['frac'], r['kernel'], 'it/traj', d['picard_iterations_per_trajectory'], 'cpu', c.get('value'), 'parity', c.get('parity_vs_gpu'))"; done
