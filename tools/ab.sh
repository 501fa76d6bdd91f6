# Interleaved A/B runs on a GPU box (gpurun -- 'bash tools/ab.sh'): in-tree builds
# paper_2603_28475_b200/libtac_{a,b}.so selected with TAC_LIB, extra environment per variant.
runt() { tag=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --tol 1e-7 --steps 16 > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err; }
for r in 1 2; do
runt cl8_$r
runt cl16_$r TAC_COMPACT_LANES=16
runt cl24_$r TAC_COMPACT_LANES=24
runt cl4_$r TAC_COMPACT_LANES=4
done
