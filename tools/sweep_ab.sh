# A/B of package copies on a few sweep cases (development aid): bash tools/sweep_ab.sh <root>...
for r in "$@"; do
  echo "== $r"
  DIFFMPC_PKG_ROOT=$r python tools/sweep.py --T 5 20 40 --B 16384 65536 --no-cpu 2>/dev/null | grep "^|" | tail -6
done
