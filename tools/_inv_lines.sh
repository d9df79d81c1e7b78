python bench.py --profile-only > gpurun_out/il_plain.log 2>&1 || exit 1
for k in yinv xinv; do
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_$k" -s 20 -c 1 -o gpurun_out/il_$k -f python bench.py --profile-only > gpurun_out/il_ncu_$k.log 2>&1
python tools/ncu_lines.py gpurun_out/il_$k.ncu-rep 45 > gpurun_out/r02h_ncu_${k}_lines.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep
