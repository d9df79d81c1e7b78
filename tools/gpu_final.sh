# final round-2 measurement: the round-2 set, the 256^3 lines and ncu --set full
# captures of every engine kernel (summaries are made from gpurun_out/ afterwards)
T=${1:-r02g}
bash tools/gpu_round2.sh $T
python bench.py --size 256 --band 64 --nt 20 --registration 0 --cpu-baseline 0 --steps 5 --warmup 3 > gpurun_out/${T}_bench_256_def.json 2>> gpurun_out/${T}_bench.err
python bench.py --size 256 --band 64 --nt 20 --registration 0 --cpu-baseline 0 --steps 5 --warmup 3 --objective state > gpurun_out/${T}_bench_256_state.json 2>> gpurun_out/${T}_bench.err
bash tools/gpu_ncu_kernels.sh ${T}k
# summaries on the box; the raw reports stay there (gpurun_out/ must stay small)
python tools/launch_summary.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launch_summary.json 2>&1
python tools/ncu_summary.py gpurun_out/${T}_dominant.ncu-rep > gpurun_out/${T}_ncu_dominant_summary.txt 2>&1
python tools/ncu_summary.py gpurun_out/${T}k_ncu_*.ncu-rep > gpurun_out/${T}_ncu_kernels_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/${T}_dominant.ncu-rep 40 > gpurun_out/${T}_ncu_dominant_lines.txt 2>&1
python tools/ncu_lines.py gpurun_out/${T}k_ncu_outer.ncu-rep 40 > gpurun_out/${T}_ncu_outer_lines.txt 2>&1
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
