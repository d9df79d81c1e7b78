# A/B of compile-time variants: every in-tree library under _lib/ (base + var_*)
# gets the GPU suite and timed GN HVPs for both objectives, interleaved twice
# so clock drift does not favour one variant.
L=paper_1807_05117_b200/_lib
libs="$L/libblreg_b200.so $(ls $L/var_*/libblreg_b200.so 2>/dev/null)"
for lib in $libs; do
  BLR_LIB_PATH=$lib python -m pytest tests -x -q -m gpu 2>&1 | tail -1 | sed "s|^|$lib: |"
done
for rep in 1 2; do
  for lib in $libs; do
    for o in deformation state; do
      BLR_LIB_PATH=$lib python bench.py --steps 40 --warmup 5 --cpu-baseline 0 --registration 0 --objective $o 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); kb=d.get('kernel_breakdown',{}); print('$rep', '$lib'.split('/')[-2], '$o', round(d['ms_per_step'],3), 'ms', 'e2e', round(d['e2e']['value'],2), 'value', round(d['value'],2), d['clocks']['sm_mhz'], ' '.join(k.replace('pad_','')+'='+str(round(v['ms'],3)) for k,v in kb.items() if v['ms']>0.5))"
    done
  done
done
