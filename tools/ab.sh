run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err; }
runt() { tag=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --tol 1e-7 --steps 16 > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err; }
for r in 1 2; do
  run a$r TAC_LIB=paper_2603_28475_b200/libtac_a.so
  run b$r TAC_LIB=paper_2603_28475_b200/libtac_b.so
done
runt tol_b TAC_LIB=paper_2603_28475_b200/libtac_b.so
runt tol_b_nocompact TAC_LIB=paper_2603_28475_b200/libtac_b.so TAC_NO_COMPACT=1
TAC_LIB=paper_2603_28475_b200/libtac_b.so timeout 1700 python -m pytest tests -m gpu -q > gpurun_out/ab_tests.log 2>&1
