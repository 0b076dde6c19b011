#!/bin/bash
# One-at-a-time sweep of the kernels' compile-time tuning macros on a GPU box: rebuilds the library with each
# setting (AXB_NVCC_EXTRA) and prints the stage-time table of tools/gpu_perf.py.  Restores the default build.
#   tools/gpu_autotune.sh > gpurun_out/autotune.log
run() {
    echo "=== $1"
    AXB_NVCC_EXTRA="$1" python -m paper_1908_05944_b200.build --force > /dev/null 2>&1 || { echo "build failed"; return; }
    python tools/gpu_perf.py 5 2>&1 | tail -4
}
run ""
for v in 2 8; do run "-DT3_WARPS_V=$v"; done
for v in 3 5; do run "-DE2_MINB=$v"; done
for v in 3 5 6 8; do run "-DPRUNE_GRID=$v"; done
for v in 2 4; do run "-DTETS_MINB=$v"; done
for v in 3 5; do run "-DPRUNE_MINB=$v"; done
for v in 1 4; do run "-DPRUNE_CLAIM_V=$v"; done
for v in 0 2; do run "-DAC2_DEPTH=$v"; done
run ""
python -m paper_1908_05944_b200.build --force > /dev/null 2>&1
