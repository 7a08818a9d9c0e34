# 1PN unstaged table loads via ld.global.ca: parity + C5 1PN kernel-time A/B against the previous library
set -x
mkdir -p gpurun_out/ldca
timeout 900 python -m pytest tests/test_gpu_extensions.py -x -q -m gpu > gpurun_out/ldca/pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/ldca/pytest.log
for rep in 1; do
for n in 64 96 128 160 200 256; do
  for lib in lib_ldca3 lib_nsrule; do
    PSWARM_LIB=tools/ab/$lib.so timeout 300 python bench.py --config c5 --nodes $n --steps 5 --warmup 3 --no-cpu-baseline \
      > gpurun_out/ldca/b_${lib}_n${n}_$rep.json 2> gpurun_out/ldca/b_${lib}_n${n}_$rep.err
  done
done
done
