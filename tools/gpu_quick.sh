# quick GPU check: parity + known answers, timed HVP for both objectives, per-category profile
python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py -x -q -m gpu 2>&1 | tail -2
for o in deformation state; do
  python bench.py --steps 30 --warmup 5 --cpu-baseline 0 --registration 0 --objective $o 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o', round(d['ms_per_step'],3), 'ms', round(d['value'],2), 'HVP/s', d['clocks'])"
  python bench.py --profile-only --objective $o 2>&1 | tail -1 > gpurun_out/prof_$o.json
done
