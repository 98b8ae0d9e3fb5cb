# per-kernel durations (ncu launch list) of base vs Gauss term arithmetic at N=32 and N=16
for v in base gauss; do
  for n in "32 8.0 2048" "16 6.0 4096"; do set -- $n
  AB_N=$1 AB_L=$2 AB_CELLS=$3 BOLTZ_LIB_VARIANT=$PWD/variants/lib_$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_conv --csv --log-file gpurun_out/ncu_${v}_$1.csv python scripts/dev/ab_step.py --child > /dev/null 2>&1
  done
done
