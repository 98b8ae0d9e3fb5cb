# N=32 joint longest-first tail (BOLTZ_LPT_TAIL_KCS) sweep, cfg5-shaped collide at 2048 cells
for t in ${TAILS:-1 2 3 4}; do
  for rep in 1 2; do
    echo "tail $t $(BOLTZ_LPT_TAIL_KCS=$t python scripts/dev/n32probe.py 2048 2>/dev/null | tail -1)"
  done
done
