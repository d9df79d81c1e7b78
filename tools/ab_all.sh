# A/B of compile-time variants (every library under _lib/: base + var_*): the GPU
# suite per library, then fp64 deformation / state and fp32 deformation GN HVPs,
# interleaved twice, with the per-category breakdown
L=paper_1807_05117_b200/_lib
libs="$L/libblreg_b200.so $(ls $L/var_*/libblreg_b200.so 2>/dev/null)"
for lib in $libs; do
  BLR_LIB_PATH=$lib python -m pytest tests -x -q -m gpu 2>&1 | tail -1 | sed "s|^|$lib: |"
done
for rep in 1 2; do
  for lib in $libs; do
    for cfg in "deformation float64" "state float64" "deformation float32"; do
      set -- $cfg
      BLR_LIB_PATH=$lib python bench.py --steps 40 --warmup 5 --cpu-baseline 0 --registration 0 --objective $1 --dtype $2 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); kb=d.get('kernel_breakdown',{}); print('$rep', '$lib'.split('/')[-2], '$1 $2', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'], ' '.join(k.replace('pad_','')+'='+str(round(v['ms'],3)) for k,v in kb.items() if v['ms']>0.5))"
    done
  done
done
