# Interleaved A/B runs on a GPU box (gpurun -- 'bash tools/ab.sh'): in-tree builds
# paper_2603_28475_b200/libtac_{a,b}.so selected with TAC_LIB, extra environment per variant.
runt() { tag=$1; shift; env "$@" timeout 600 python bench.py --no-cpu-baseline --tol 1e-7 --steps 16 > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err; }
for r in 1 2; do
runt rb256_$r TAC_REMAP_BLOCKS=256
runt rb384_$r TAC_REMAP_BLOCKS=384
runt rb512_$r TAC_REMAP_BLOCKS=512
runt rb768_$r TAC_REMAP_BLOCKS=768
done
