# k_conv_mirror2<16> (the default N=16 collide/RK2 K2 since round 2): bench line, launch list and one --set full capture
set -e
mkdir -p gpurun_out/r2m
python bench.py --steps 20 --warmup 5 > gpurun_out/r2m/bench.json 2> gpurun_out/r2m/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2m/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-n32 --no-cfg3 --no-cpu-baseline > /dev/null 2>&1
AB_N=16 AB_L=6.0 AB_CELLS=4096 ncu --set full --import-source on --clock-control none -k regex:k_conv_mirror2 -s 2 -c 1 \
    -o gpurun_out/r2m/mirror2_16 python scripts/dev/ab_step.py --child > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/r2m/mirror2_16.ncu-rep > gpurun_out/r2m/mirror2_16_ncu.txt 2>&1 || true
