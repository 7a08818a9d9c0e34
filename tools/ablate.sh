# Diagnostic builds of the library with one phase of k_pc_ws removed (results invalid):
# 1 = no MMA epilogue (main rows), 2 = no force, 3 = no DMMA, 4 = no b0 GEMV, 5 = folded operator loads
# L1-hot (k-pair 0 only), 6 = folded B fragments from k-steps 0-1 only.  Timing only (tools/probe_phases.py).
# usage: bash tools/ablate.sh [modes...]  (default 1 2 3 4 5 6)
set -e
cd "$(dirname "$0")/../paper_2301_03989_b200/csrc"
for k in ${@:-1 2 3 4 5 6}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr \
    -I../../include -I. -DPSWARM_ABLATE=$k -c pc_slots2.cu -o /tmp/pc_slots2_ablate$k.o &
done
wait
for k in ${@:-1 2 3 4 5 6}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../tools/ab/lib_ablate$k.so \
    pc_kernels.o /tmp/pc_slots2_ablate$k.o pc_rk.o pswarm_capi.o
done
