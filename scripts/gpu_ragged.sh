mkdir -p gpurun_out
for w in decode_configs3 decode_ragged_configs3; do
  timeout 600 ncu --set full --clock-control none -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/prof_${w} -f python scripts/prof_kernels.py $w 4 > /dev/null 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_${w}.ncu-rep > gpurun_out/sum_${w}.txt 2>&1
  python scripts/sass_stalls.py gpurun_out/prof_${w}.ncu-rep 12 > gpurun_out/stalls_${w}.txt 2>&1
  ncu -i gpurun_out/prof_${w}.ncu-rep --page details --csv 2>/dev/null | grep -iE 'Achieved Occupancy|Theoretical Occupancy|Block Limit|Waves Per SM|Registers Per|Grid Size|Duration|DRAM Throughput|L2 Hit|Mem Busy|Max Bandwidth' > gpurun_out/det_${w}.txt
done
rm -f gpurun_out/*.ncu-rep
cat gpurun_out/sum_decode*.txt gpurun_out/det_decode*.txt
