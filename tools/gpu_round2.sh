# round-2 measurement set: GPU suite, default bench (+ reference arm sample),
# state / fp32 / batch lines, launch list, ncu --set full of the dominant kernel
T=${1:-r02}
python -m pytest tests -q -m gpu > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "suite rc=$?"; tail -2 gpurun_out/${T}_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${T}_smoke.log
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
python bench.py --objective state --registration 0 --cpu-baseline 0 > gpurun_out/${T}_bench_state.json 2>> gpurun_out/${T}_bench.err
python bench.py --dtype float32 --registration 0 --cpu-baseline 0 > gpurun_out/${T}_bench_f32.json 2>> gpurun_out/${T}_bench.err
python bench.py --batch 64 > gpurun_out/${T}_bench_batch64.json 2>> gpurun_out/${T}_bench.err
python bench.py --steps 2 --warmup 3 --registration 0 --cpu-baseline 0 > gpurun_out/${T}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 2 --warmup 3 --registration 0 --cpu-baseline 0 > gpurun_out/${T}_ncu_launch.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:int\)2>\(blr::LineArgs" -s 4 -c 1 \
    -o gpurun_out/${T}_dominant -f python bench.py --profile-only > gpurun_out/${T}_ncu_full.log 2>&1; echo "ncu full rc=$?"
