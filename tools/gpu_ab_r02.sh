# same-box A/B: this build vs the round-2 baseline build (tools/ab/lib_r02base.so)
bash tools/probe_ab_lib.sh tools/ab/lib_r02base.so 2>&1 | grep -v "^$"
