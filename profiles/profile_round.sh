#!/bin/bash
# One profiling pass of the current build on a GPU box (gpurun from the repo root: profiles/profile_round.sh):
#   1. the default bench line (with cpu_baseline) -> gpurun_out/prof_bench.json
#   2. the ncu launch list of one timed step (cold-cache, serialised) -> gpurun_out/prof_launches.csv
#   3. ncu --set full of each main kernel mid-trajectory -> gpurun_out/prof_full.ncu-rep
set -e
python bench.py > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err
python bench.py --steps 1 --warmup 4 --no-cpu-baseline > gpurun_out/prof_plain.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 3400 -c 900 --csv \
    --log-file gpurun_out/prof_launches.csv python bench.py --steps 1 --warmup 4 --no-cpu-baseline \
    > gpurun_out/prof_launches.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"elem_grad_rows|elem_grad_cells|elem_curv_cells|classify|k_contact_near|friction|curv_direct|vert_pre|dir_apply|dir_reduce|broadphase_list" \
    -s 2000 -c 12 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 4 --no-cpu-baseline \
    > gpurun_out/prof_full.log 2>&1
echo profile-done
