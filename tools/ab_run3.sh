export AB_ONLY=${AB_ONLY:-quad13-f32-d}
for r in 1 2; do for v in $AB_VARIANTS; do python tools/ab_bench.py ab/$v 20 2>&1 | grep -v Warn; done; done
