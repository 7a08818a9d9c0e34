# force_pair body-loop unroll (PSWARM_FP_UNROLL 1..4) A/B: C4 and Newtonian C5 legs, kernel time
mkdir -p gpurun_out/unroll
for rep in 1 2; do
  for lib in lib_u1 lib_u2 lib_u3 lib_u4; do
    PSWARM_LIB=tools/ab/$lib.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/unroll/c4_${lib}_$rep.json 2>/dev/null
    for n in 128 160 256; do
      PSWARM_LIB=tools/ab/$lib.so timeout 300 python bench.py --config c5 --nodes $n --force n_body --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/unroll/n${n}_${lib}_$rep.json 2>/dev/null
    done
  done
done
