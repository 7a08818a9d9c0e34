# 1PN accumulator merge: parity tests + C5 1PN kernel-time A/B against the previous library
set -x
mkdir -p gpurun_out/relacc
timeout 900 python -m pytest tests/test_gpu_extensions.py tests/test_gpu_propagate.py -x -q -m gpu > gpurun_out/relacc/pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/relacc/pytest.log
for rep in 1 2; do
for n in 64 128 200 256; do
  for lib in lib_pre_relacc lib_relacc; do
    PSWARM_LIB=tools/ab/$lib.so timeout 300 python bench.py --config c5 --nodes $n --steps 5 --warmup 3 --no-cpu-baseline \
      > gpurun_out/relacc/b_${lib}_n${n}_$rep.json 2> gpurun_out/relacc/b_${lib}_n${n}_$rep.err
  done
done
done
