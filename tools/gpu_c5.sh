# GPU tests + C5 node sweep (relativistic) + C2 probe
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for n in 64 96 128 200; do
  timeout 600 python bench.py --config c5 --nodes $n --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c5_n$n.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bench_c5_n$n.json')); print($n, d['value'], d['roofline']['frac'])"
done
for n in 64 128; do
  timeout 600 python bench.py --config c4 --per-gpu 100000 --nodes $n --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_nb_n$n.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bench_nb_n$n.json')); print('newton', $n, d['value'], d['roofline']['frac'])"
done
python tools/probe_perf.py | head -1
