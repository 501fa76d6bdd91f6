run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err; }
runt() { tag=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --tol 1e-7 --steps 16 > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err; }
for v in a b; do TAC_LIB=paper_2603_28475_b200/libtac_$v.so timeout 600 python tools/diag_tail.py --only-1024 --reps 2 --n-active 1 > gpurun_out/ab_tail_${v}_1.log 2>&1; done
for r in 1 2; do
  run a$r TAC_LIB=paper_2603_28475_b200/libtac_a.so
  run b$r TAC_LIB=paper_2603_28475_b200/libtac_b.so
done
runt tol_a TAC_LIB=paper_2603_28475_b200/libtac_a.so
runt tol_b TAC_LIB=paper_2603_28475_b200/libtac_b.so
TAC_LIB=paper_2603_28475_b200/libtac_b.so timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py -q -x > gpurun_out/ab_tests.log 2>&1
