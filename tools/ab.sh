# Interleaved A/B runs on a GPU box (gpurun -- 'bash tools/ab.sh'): in-tree builds
# paper_2603_28475_b200/libtac_{a,b,c}.so selected with TAC_LIB, extra environment per variant.
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err; }
for r in 1 2; do
  run base$r
  run body$r TAC_CLS_BODY=1
done
