# usage: LIB=name ENVS="A=1 B=2+C=3" bash tools/ab_env.sh  (one stage_bench per setting; '+' joins variables)
for e in "" $ENVS; do for c in ${CONFIGS:-C3 C5 C2}; do env ${e//+/ } SNP_LIB_PATH=abtest/libsnp_$LIB.so python tools/stage_bench.py --config $c --iters 40 2>&1 | sed "s/.n_visible.*overflow_pixels/ ovf/" | sed "s/^/$LIB [$e] /"; done; done
