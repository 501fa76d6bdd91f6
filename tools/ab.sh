runt() { tag=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --tol 1e-7 --steps 16 > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err; }
for na in 1 8; do
  for v in a b; do
    TAC_LIB=paper_2603_28475_b200/libtac_$v.so timeout 600 python tools/diag_tail.py --only-1024 --reps 2 --n-active $na > gpurun_out/ab_tail_${v}_$na.log 2>&1
  done
done
runt tol_a TAC_LIB=paper_2603_28475_b200/libtac_a.so
runt tol_b TAC_LIB=paper_2603_28475_b200/libtac_b.so
TAC_LIB=paper_2603_28475_b200/libtac_b.so timeout 900 python -m pytest tests/test_gpu_api.py -q -k "tolerance or remap or sharded" > gpurun_out/ab_tests.log 2>&1
