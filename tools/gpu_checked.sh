# bounds-checked library (BLR_CHECKED=1): full GPU suite, the fused forward pass
# on, and the large engine lengths; any violated BLR_CHECK traps with its tag
L=paper_1807_05117_b200/_lib/var_checked/libblreg_b200.so
T=${1:-r02}
BLR_LIB_PATH=$L timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${T}_checked_pytest.log 2>&1; echo "suite rc=$?"; tail -2 gpurun_out/${T}_checked_pytest.log
BLR_FWD2=1 BLR_LIB_PATH=$L timeout 1500 python -m pytest tests -q -m gpu -k "parity or headline or solver or fused" > gpurun_out/${T}_checked_pytest_fused.log 2>&1; echo "fused rc=$?"; tail -2 gpurun_out/${T}_checked_pytest_fused.log
for c in small l100 l196; do
  BLR_LIB_PATH=$L timeout 900 python tools/sanitize_smoke.py $c > gpurun_out/${T}_checked_smoke_$c.log 2>&1; echo "smoke $c rc=$?"
  BLR_LIB_PATH=$L timeout 900 python tools/sanitize_smoke.py $c --fused > gpurun_out/${T}_checked_smoke_${c}_fused.log 2>&1; echo "smoke $c fused rc=$?"
done
grep -h "BLR_CHECK" gpurun_out/${T}_checked_*.log | head; echo "checks-fired: $(grep -h BLR_CHECK gpurun_out/${T}_checked_*.log | wc -l)"
