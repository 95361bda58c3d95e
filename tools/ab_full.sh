# full snp_render A/B (K5 + K6w + K6) of library variants, 3 interleaved rounds:
# VARIANTS="a b ..." CFGS="C3 C5" bash tools/ab_full.sh
for r in 1 2 3; do for v in $VARIANTS; do for c in ${CFGS:-C3 C5}; do
  L=abtest/libsnp_$v.so; [ "$v" = cur ] && L=paper_2510_08491_b200/libsnp.so
  SNP_LIB_PATH=$L python tools/stage_bench.py --config $c --iters ${ITERS:-30} 2>&1 | tail -1 | \
    sed -n "s/.*'bin_sort': \([0-9.]*\), 'render': \([0-9.]*\).*/$v $c \2 \1/p"
done; done; done
