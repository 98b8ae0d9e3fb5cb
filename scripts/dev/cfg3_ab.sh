# cfg3 (Nx=256 Strang steps, latency schedule, CUDA graph) A/B over library variants
for rep in 1 2; do
  for v in "$@"; do
    echo "$(basename $v) $(BOLTZ_LIB_VARIANT=$(realpath $v) python scripts/run_config.py --config 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4))')"
  done
done
