#!/bin/bash
# End-of-round measurements of the current build (gpurun from the repo root): GPU tests, smoke,
# the other workloads and modes; then profiles/profile_round.sh (default bench line + ncu).
T=${TAG:-vX}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/fin_gpu_tests_$T.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke_$T.log 2>&1
for c in c5 c3u c2 c1; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/fin_bench_${c}_$T.json 2>/dev/null; done
timeout 600 python bench.py --iters 100 --no-cpu-baseline > gpurun_out/fin_bench_k100_$T.json 2>/dev/null
timeout 900 python bench.py --tol 1e-7 --steps 16 --no-cpu-baseline > gpurun_out/fin_bench_tol_$T.json 2>/dev/null
timeout 900 python bench.py --tol 1e-7 --steps 16 --max-iters 600 --no-cpu-baseline > gpurun_out/fin_bench_tol600_$T.json 2>/dev/null
timeout 900 python bench.py --tol 1e-7 --steps 16 --max-iters 300 --no-cpu-baseline > gpurun_out/fin_bench_tol300_$T.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin_bench_ref_$T.json 2>/dev/null
bash profiles/profile_round.sh > gpurun_out/fin_prof_$T.log 2>&1
echo final-done
