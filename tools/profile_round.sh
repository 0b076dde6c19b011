#!/bin/bash
# One profiling round on the GPU box: bench line, ncu launch list of the same command, ncu --set full of the hot kernels.
#   tools/profile_round.sh <tag>      (outputs under gpurun_out/<tag>_*)
tag=${1:-round}
mkdir -p gpurun_out
python bench.py --steps 100 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_reference_arm.json 2>> gpurun_out/${tag}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_bench_1M_a0.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${tag}_launches.log 2>&1
ncu --set full --import-source on --clock-control none \
    -k regex:"k_edges|k_tri_tet3|k_prune_tris|k_prune_tets|k_prune_edges|k_cell_finalize|k_scatter_edges_tris|k_emit_tris|k_scan_lookback" \
    --launch-skip 10 -c 10 -o gpurun_out/${tag}_full python tools/one_step.py 1000000 0 2 > gpurun_out/${tag}_full.log 2>&1
ncu -i gpurun_out/${tag}_full.ncu-rep --page raw --csv > gpurun_out/${tag}_ncu_full_raw.csv 2>/dev/null
cat gpurun_out/${tag}_bench.json
ncu --set full --clock-control none -k regex:"k_edges|k_tri_tet3|k_prune_tris|k_prune_tets|k_prune_edges|k_scatter_edges_tris|k_emit_tris" \
    --launch-skip 7 -c 7 -o gpurun_out/${tag}_a14_full python tools/one_step.py 1000000 1.4 2 > gpurun_out/${tag}_a14_full.log 2>&1
ncu -i gpurun_out/${tag}_a14_full.ncu-rep --page raw --csv > gpurun_out/${tag}_a14_ncu_full_raw.csv 2>/dev/null
