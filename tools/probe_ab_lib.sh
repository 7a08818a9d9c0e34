# A/B of two builds of the library on one box (diagnostics): kernel time of the folded
# kernel at N = 200 / 160, interleaved runs.  usage: bash tools/probe_ab_lib.sh OTHER.so
for rep in 1 2; do
  for lib in paper_2301_03989_b200/libpswarm_b200.so "$1"; do
    echo "== $lib"; PSWARM_LIB=$lib python tools/probe_ab.py fast_decide 1 1 20000 200 | head -1
    PSWARM_LIB=$lib python tools/probe_ab.py fast_decide 1 1 1000 200 | head -1
    PSWARM_LIB=$lib python tools/probe_ab.py fast_decide 1 1 20000 160 | head -1
  done
done
