for r in 1 2; do
  (cd abtest_old && timeout 200 python scripts/epi_matrix.py 4096 1000 | sed 's/^/old: /')
  timeout 200 python scripts/epi_matrix.py 4096 1000 | sed 's/^/new: /'
done
