# A/B of the config-5 step on one box: the tree in abtest_old/ (a previous
# build) vs the working tree, alternated, same process settings.
B=${1:-65536}
for r in 1 2; do
  (cd abtest_old && timeout 200 python scripts/step_gemms.py --batch $B --steps 10 | head -1 | sed 's/^/old: /')
  timeout 200 python scripts/step_gemms.py --batch $B --steps 10 | head -1 | sed 's/^/new: /'
done
