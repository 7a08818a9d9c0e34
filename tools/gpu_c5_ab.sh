# 1PN (C5) kernel-time A/B against the round-2 baseline build + the GPU suite (diagnostics)
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for n in 64 128 200; do
  for lib in paper_2301_03989_b200/libpswarm_b200.so tools/ab/lib_r02base.so; do
    PSWARM_LIB=$lib timeout 300 python bench.py --config c5 --nodes $n --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$n', '$lib'.split('/')[-1], d['value'], r['kernel_ms'], r['frac'], r['kernel'])"
  done
done
