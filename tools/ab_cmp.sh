# A/B of library variants: VARIANTS="base new ..." (abtest/libsnp_<v>.so; "cur" = the in-tree build)
set -e
CFGS=${CFGS:-"C3 C5 C2"}
for r in 1 2; do for v in $VARIANTS; do for c in $CFGS; do
  if [ "$v" = cur ]; then L=paper_2510_08491_b200/libsnp.so; else L=abtest/libsnp_$v.so; fi
  SNP_LIB_PATH=$L python tools/stage_bench.py --config $c --iters ${ITERS:-40} 2>&1 | tail -1 | sed "s/^/$v /" | cut -c1-140
done; done; done
