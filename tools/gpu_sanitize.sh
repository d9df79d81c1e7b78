# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_smoke.py;
# logs under gpurun_out/ (summaries copied to profiles/ by hand)
CS="compute-sanitizer --error-exitcode 9 --print-limit 50"
T=${1:-r02}
timeout 900 $CS --tool memcheck python tools/sanitize_smoke.py small > gpurun_out/${T}_san_memcheck_small.log 2>&1; echo "memcheck small rc=$?"
timeout 900 $CS --tool memcheck python tools/sanitize_smoke.py small --fused > gpurun_out/${T}_san_memcheck_small_fused.log 2>&1; echo "memcheck small fused rc=$?"
timeout 1500 $CS --tool memcheck python tools/sanitize_smoke.py l100 > gpurun_out/${T}_san_memcheck_l100.log 2>&1; echo "memcheck l100 rc=$?"
timeout 1500 $CS --tool memcheck python tools/sanitize_smoke.py l196 > gpurun_out/${T}_san_memcheck_l196.log 2>&1; echo "memcheck l196 rc=$?"
timeout 1500 $CS --tool racecheck --racecheck-report hazard python tools/sanitize_smoke.py small > gpurun_out/${T}_san_racecheck_small.log 2>&1; echo "racecheck small rc=$?"
timeout 1500 $CS --tool racecheck --racecheck-report hazard python tools/sanitize_smoke.py small --fused > gpurun_out/${T}_san_racecheck_small_fused.log 2>&1; echo "racecheck small fused rc=$?"
timeout 1500 $CS --tool synccheck python tools/sanitize_smoke.py small > gpurun_out/${T}_san_synccheck_small.log 2>&1; echo "synccheck small rc=$?"
timeout 1500 $CS --tool synccheck python tools/sanitize_smoke.py small --fused > gpurun_out/${T}_san_synccheck_small_fused.log 2>&1; echo "synccheck small fused rc=$?"
timeout 2400 $CS --tool racecheck --racecheck-report hazard python tools/sanitize_smoke.py l100 > gpurun_out/${T}_san_racecheck_l100.log 2>&1; echo "racecheck l100 rc=$?"
tail -n 3 gpurun_out/${T}_san_*.log
