#!/bin/bash
# A/B builds on the GPU box: tools/ab.sh "<nvcc extra flags>" ... ; each variant is built and timed with gpu_perf.py
for v in "$@"; do
  echo "=== variant: $v"
  AXB_NVCC_EXTRA="$v" python -m paper_1908_05944_b200.build --force > /dev/null || exit 1
  python tools/gpu_perf.py ${REPS:-10} 2>&1 | cut -c1-14,56-200
done
