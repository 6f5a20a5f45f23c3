export AB_ONLY=${AB_ONLY:-quad13-f32}
for r in a0 a1 a0 a1; do python tools/ab_bench.py ab/$r 20 2>&1 | grep -v Warn; done
