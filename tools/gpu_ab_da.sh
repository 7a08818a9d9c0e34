# decision arguments in shared memory vs kernel parameters: C4 + C5 legs kernel time, phase counters
mkdir -p gpurun_out/da
for rep in 1 2; do
  for lib in lib_base lib_da; do
    PSWARM_LIB=tools/ab/$lib.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/da/c4_${lib}_$rep.json 2>/dev/null
    for c in "--nodes 64 --force n_body" "--nodes 128 --force n_body" "--nodes 200 --force n_body" "--nodes 96" "--nodes 200"; do
      tag=$(echo $c | tr -d ' -')
      PSWARM_LIB=tools/ab/$lib.so timeout 300 python bench.py --config c5 $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/da/${tag}_${lib}_$rep.json 2>/dev/null
    done
  done
done
for lib in lib_base lib_da; do
  PSWARM_LIB=tools/ab/$lib.so timeout 300 python tools/probe_phases.py 20000 planets8 64 > gpurun_out/da/ph64_$lib.json 2>/dev/null
  PSWARM_LIB=tools/ab/$lib.so timeout 300 python tools/probe_phases.py 20000 planets8 200 > gpurun_out/da/ph200_$lib.json 2>/dev/null
done
