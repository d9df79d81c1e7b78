# Stage the reference's own tests and probe (unmodified) into the git-ignored
# baseline/_ref_tests/ so the GPU box can run them against the numpy-facing
# compat layer (tests/test_gpu_reference_suite.py).  Run in the build
# container, where /root/reference exists; nothing here enters git history.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
DST=$ROOT/baseline/_ref_tests
rm -rf "$DST"; mkdir -p "$DST/tests"
cp /root/reference/pkg/tests/helpers.py /root/reference/pkg/tests/test_objectives.py \
   /root/reference/pkg/tests/test_solver.py /root/reference/pkg/tests/test_spectral.py \
   /root/reference/pkg/tests/test_transport.py "$DST/tests/"
cp /root/reference/pkg/probe_hvp.py "$DST/"
echo "staged $(ls "$DST/tests" | wc -l) test files into $DST"
