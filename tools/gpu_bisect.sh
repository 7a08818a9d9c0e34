# same-box kernel-time comparison of several library builds (diagnostics)
# usage: bash tools/gpu_bisect.sh LIB...   (the in-tree build is always measured first)
for rep in 1 2; do
  for lib in paper_2301_03989_b200/libpswarm_b200.so "$@"; do
    echo "$lib $(PSWARM_LIB=$lib python tools/probe_ab.py fast_decide 1 1 20000 200 | head -1)"
  done
done
