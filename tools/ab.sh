set -e
for r in 1 2; do for v in $VARIANTS; do for c in C3 C5 C2; do SNP_LIB_PATH=abtest/libsnp_$v.so python tools/stage_bench.py --config $c --iters 40 2>&1 | sed "s/^/$v /" ; done; done; done
