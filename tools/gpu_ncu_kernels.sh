# ncu --set full captures of the engine kernels named on the command line
# (default: the ones VERDICT r1 asked to re-capture).  Usage on the box:
#   bash tools/gpu_ncu_kernels.sh TAG [objective]
TAG=${1:-r02}
OBJ=${2:-deformation}
mkdir -p gpurun_out
python bench.py --profile-only --objective $OBJ > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/${TAG}_plain.log; exit 1; }
cap() {  # name regex skip
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$2" -s $3 -c 1 -o gpurun_out/${TAG}_ncu_$1 -f \
    python bench.py --profile-only --objective $OBJ > gpurun_out/${TAG}_ncu_$1.log 2>&1
  echo "ncu $1 rc=$?"
}
cap outer    'int\)6>\(blr::LineArgs' 4
cap map_tc   'int\)2>\(blr::LineArgs' 4
cap yfwd     'k_yfwd' 20
cap xfwd     'k_xfwd' 20
cap yinv     'k_yinv' 20
cap xinv     'k_xinv' 20
