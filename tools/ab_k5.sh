# K5-only A/B (SNP_DEBUG=2: K6w/K6 skipped) of library variants over configs, 3 rounds
# interleaved: VARIANTS="a b ..." CFGS="C3 C5" bash tools/ab_k5.sh
for r in 1 2 3; do for v in $VARIANTS; do for c in ${CFGS:-C3 C5}; do
  L=abtest/libsnp_$v.so; [ "$v" = cur ] && L=paper_2510_08491_b200/libsnp.so
  SNP_DEBUG=2 SNP_LIB_PATH=$L python tools/stage_bench.py --config $c --iters ${ITERS:-30} 2>&1 | tail -1 | \
    sed -n "s/.*'render': \([0-9.]*\).*/$v $c \1/p"
done; done; done
