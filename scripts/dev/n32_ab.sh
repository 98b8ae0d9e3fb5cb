# N=32 collide A/B over library variants (BOLTZ_LIB_VARIANT), cfg5-shaped, 2048 cells
for rep in 1 2; do
  for v in "$@"; do
    echo "$(basename $v) $(BOLTZ_LIB_VARIANT=$(realpath $v) python scripts/dev/n32probe.py 2048 2>/dev/null | tail -1)"
  done
done
