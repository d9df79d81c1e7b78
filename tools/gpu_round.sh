# round artifacts: full GPU tests, default bench (+reference arm), launch list, ncu of the dominant kernel
set -x
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --objective state --registration 0 --cpu-baseline 0 > gpurun_out/bench_state.json 2>> gpurun_out/bench.err
python bench.py --dtype float32 --registration 0 --cpu-baseline 0 > gpurun_out/bench_f32.json 2>> gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.json 2>> gpurun_out/bench.err
python bench.py --steps 2 --warmup 3 --registration 0 --cpu-baseline 0 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --registration 0 --cpu-baseline 0 > gpurun_out/ncu_launch.log 2>&1
python bench.py --profile-only > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:int\)2>\(blr::LineArgs" -s 2 -c 1 -o gpurun_out/dominant python bench.py --profile-only > gpurun_out/ncu_full.log 2>&1
echo done
