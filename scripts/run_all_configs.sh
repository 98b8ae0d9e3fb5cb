# BASELINE configs 1-5 on one B200 (cfg4 with hard spheres and Maxwell molecules,
# cfg3 also with the SPEC single-stage transport); one JSON line per run
set -e
out=${1:-gpurun_out/configs.jsonl}
: > $out
python scripts/run_config.py --config 1 >> $out
python scripts/run_config.py --config 2 >> $out
python scripts/run_config.py --config 3 >> $out
python scripts/run_config.py --config 3 --transport single_stage >> $out
python scripts/run_config.py --config 4 --lam 1 >> $out
python scripts/run_config.py --config 4 --lam 0 >> $out
python scripts/run_config.py --config 5 >> $out
