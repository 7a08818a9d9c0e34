# FP-group first-iteration flags as a register bitmask instead of a local bool array: Newtonian A/B
set -x
mkdir -p gpurun_out/firstm
for rep in 1 2 3; do
for cfgs in "c5 --nodes 200 --force n_body" "c5 --nodes 128 --force n_body" "c5 --nodes 256 --force n_body"; do
  tag=$(echo $cfgs | tr ' ' '_')
  for lib in lib_ldca3 lib_firstm; do
    PSWARM_LIB=tools/ab/$lib.so timeout 300 python bench.py --config $cfgs --steps 5 --warmup 3 --no-cpu-baseline \
      > gpurun_out/firstm/b_${lib}_${tag}_$rep.json 2> /dev/null
  done
done
done
