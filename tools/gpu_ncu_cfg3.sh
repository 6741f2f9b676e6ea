# GPU-box session: cfg3 A/B (TMA columns on/off) + ncu --set full with source of all three cfg3 kernels.
mkdir -p gpurun_out
timeout 300 python tools/ab.py cfg3 HK_NO_COLTMA=1 "" > gpurun_out/ab3.txt 2>&1
python tools/cfg.py cfg3 1 > /dev/null
for i in 0 1 2; do
  timeout 600 ncu --set full --clock-control none --import-source on -s $((3+i)) -c 1 -o gpurun_out/k$i python tools/cfg.py cfg3 1 > /dev/null 2>&1
  ncu -i gpurun_out/k$i.ncu-rep --page raw --csv > gpurun_out/k${i}_raw.csv 2>/dev/null
  ncu -i gpurun_out/k$i.ncu-rep --page source --csv > gpurun_out/k${i}_source.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep
