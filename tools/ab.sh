run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err; }
for r in 1 2; do
  run base$r TAC_LIB=paper_2603_28475_b200/libtac_b.so
  run anc4_$r TAC_LIB=paper_2603_28475_b200/libtac_b.so TAC_ANC_NB=4
  run anc16_$r TAC_LIB=paper_2603_28475_b200/libtac_b.so TAC_ANC_NB=16
  run bp16k_$r TAC_LIB=paper_2603_28475_b200/libtac_b.so TAC_BP_BLOCKS=16384
  run bp2k_$r TAC_LIB=paper_2603_28475_b200/libtac_b.so TAC_BP_BLOCKS=2368
done
