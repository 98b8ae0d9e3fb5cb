# End-of-round evidence on one B200: the default bench line, its ncu launch list, and
# --set full summaries of the N=16 K2 (k_conv_mirror2), the line K1/K3, and the N=32 kernels
# (SKIP_BENCH=1: the launch lists and captures only)
set -e
out=${OUT:-gpurun_out/final}; mkdir -p $out
[ -n "$SKIP_BENCH" ] || python bench.py --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-n32 --no-cfg3 --no-cpu-baseline > /dev/null 2>&1
AB_N=16 AB_L=6.0 AB_CELLS=4096 ncu --set full --import-source on --clock-control none -k regex:"k_conv_mirror2|_line" -s 4 -c 4 \
    -o $out/n16 python scripts/dev/ab_step.py --child > /dev/null 2>&1
python scripts/ncu_summary.py $out/n16.ncu-rep > $out/n16_ncu.txt 2>&1 || true
AB_N=32 AB_L=8.0 AB_CELLS=2048 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_conv" -c 20 --csv \
    --log-file $out/n32_launches.csv python scripts/dev/ab_step.py --child > /dev/null 2>&1
AB_N=32 AB_L=8.0 AB_CELLS=512 ncu --set full --import-source on --clock-control none -k regex:"k_conv_kcs" -s 5 -c 5 \
    -o $out/n32 python scripts/dev/ab_step.py --child > /dev/null 2>&1
python scripts/ncu_summary.py $out/n32.ncu-rep > $out/n32_ncu.txt 2>&1 || true
rm -f $out/n16.ncu-rep
[ -n "$SKIP_BENCH" ] || python scripts/run_config.py --config 1 > $out/cfg1.json
ls -la $out
