# cfg1 (one cell) A/B over library variants: K2 cell schedule, 50 RK2 steps as graph replays
for rep in 1 2; do
  for v in "$@"; do
    echo "$(basename $v) $(BOLTZ_LIB_VARIANT=$(realpath $v) python scripts/dev/cfg1_time.py cell 2>/dev/null | tr '\n' ' ')"
  done
done
