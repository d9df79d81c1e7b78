L=paper_1807_05117_b200/_lib
for lib in $L/libblreg_b200.so $L/var_tw0/libblreg_b200.so; do
  BLR_LIB_PATH=$lib python -m pytest tests -x -q -m gpu 2>&1 | tail -1 | sed "s|^|$lib: |"
done
for rep in 1 2; do
  for lib in $L/libblreg_b200.so $L/var_tw0/libblreg_b200.so; do
    for o in deformation state; do
      BLR_LIB_PATH=$lib python bench.py --steps 40 --warmup 5 --cpu-baseline 0 --registration 0 --objective $o --dtype float32 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$rep', '$lib'.split('/')[-2], '$o f32', round(d['ms_per_step'],3), 'ms', 'value', round(d['value'],2), d['clocks']['sm_mhz'])"
    done
  done
done
