# A/B of package copies ab/a0.. with per-copy env (development aid)
export AB_ONLY=${AB_ONLY:-quad13-f32-dense}
for r in 1 2; do
python tools/ab_bench.py ab/a0 20 2>&1 | grep -v Warn
python tools/ab_bench.py ab/a1 20 2>&1 | grep -v Warn
DIFFMPC_GPB=2 python tools/ab_bench.py ab/a2 20 2>&1 | grep -v Warn
DIFFMPC_GPB=2 python tools/ab_bench.py ab/a3 20 2>&1 | grep -v Warn
done
