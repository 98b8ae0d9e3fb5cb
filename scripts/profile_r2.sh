# Round-2 evidence on one B200: the default bench line, its ncu launch list,
# and --set full captures of the dominant kernels (N=16 K2 mirror, N=32 kcsr
# REST, the N=16 line K3) -- each ncu pass after its program exited 0 without ncu
set -e
mkdir -p gpurun_out/r2
python bench.py --steps 20 --warmup 5 > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-n32 --no-cfg3 --no-cpu-baseline > /dev/null 2>&1
AB_N=16 AB_L=6.0 AB_CELLS=4096 ncu --set full --import-source on --clock-control none -k regex:k_conv_mirror -s 2 -c 1 \
    -o gpurun_out/r2/mirror16 python scripts/dev/ab_step.py --child > /dev/null 2>&1
AB_N=16 AB_L=6.0 AB_CELLS=4096 ncu --set full --import-source on --clock-control none -k regex:k_inv_line -s 2 -c 2 \
    -o gpurun_out/r2/invline16 python scripts/dev/ab_step.py --child > /dev/null 2>&1
AB_N=32 AB_L=8.0 AB_CELLS=512 ncu --set full --import-source on --clock-control none -k regex:"k_conv_kcs" -s 5 -c 5 \
    -o gpurun_out/r2/kcsm32 python scripts/dev/ab_step.py --child > /dev/null 2>&1
AB_N=32 AB_L=8.0 AB_CELLS=2048 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_conv" -c 20 --csv \
    --log-file gpurun_out/r2/kcsm32_launches.csv python scripts/dev/ab_step.py --child > /dev/null 2>&1
for r in mirror16 invline16 kcsm32; do
  python scripts/ncu_summary.py gpurun_out/r2/$r.ncu-rep > gpurun_out/r2/${r}_ncu.txt 2>&1 || true
done
rm -f gpurun_out/r2/invline16.ncu-rep gpurun_out/r2/kcsm32.ncu-rep   # keep the merge-back under 64 MiB
ls -la gpurun_out/r2
