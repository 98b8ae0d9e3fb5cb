# K2 term arithmetic A/B: default 6-instruction term vs the Gauss 5-instruction form
for n in "16 6.0 4096" "24 8.0 1024" "32 8.0 2048"; do set -- $n
  echo "N=$1 cells=$3"
  AB_N=$1 AB_L=$2 AB_CELLS=$3 python scripts/dev/ab_step.py variants/lib_base.so variants/lib_gauss.so
done
