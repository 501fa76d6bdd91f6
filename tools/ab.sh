run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err; }
runt() { tag=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --tol 1e-7 --steps 16 > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err; }
for r in 1 2; do
  run a$r TAC_LIB=paper_2603_28475_b200/libtac_a.so
  run b$r TAC_LIB=paper_2603_28475_b200/libtac_b.so
done
runt tol_b TAC_LIB=paper_2603_28475_b200/libtac_b.so
TAC_LIB=paper_2603_28475_b200/libtac_b.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -x > gpurun_out/ab_tests.log 2>&1
