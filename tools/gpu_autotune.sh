#!/bin/bash
# One-at-a-time sweep of the kernels' compile-time tuning macros on a GPU box: rebuilds the library with each
# setting (AXB_NVCC_EXTRA) and prints the stage-time table of tools/gpu_perf.py.  Restores the default build.
#   tools/gpu_autotune.sh "<flags 1>" "<flags 2>" ... > gpurun_out/autotune.log
run() {
    echo "=== $1"
    AXB_NVCC_EXTRA="$1" python -m paper_1908_05944_b200.build --force > /dev/null 2>&1 || { echo "build failed"; return; }
    python tools/gpu_perf.py 5 2>&1 | tail -4
}
run ""
for f in "$@"; do run "$f"; done
run ""
python -m paper_1908_05944_b200.build --force > /dev/null 2>&1
