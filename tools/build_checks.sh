#!/bin/bash
# build_checks.sh: libgs.so with the device-side bounds checks (-DGS_CHECKS, see
# gs_common.cuh GS_DCHECK) at paper_2507_15683_b200/_build/checks/libgs.so;
# load it with GS_LIB=... (compute-sanitizer is closed on the GPU pool).
set -e
cd "$(dirname "$0")/.."
B=paper_2507_15683_b200/_build/checks; mkdir -p $B
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I include -ftz=false -prec-div=true -prec-sqrt=true --expt-relaxed-constexpr -DGS_CHECKS"
objs=""
for f in paper_2507_15683_b200/csrc/*.cu; do
  n=$(basename $f .cu); extra=""
  [ "$n" == "gs_project" ] && extra="-fmad=false"
  nvcc $F $extra -c $f -o $B/$n.o &
  objs="$objs $B/$n.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $B/libgs.so $objs -lcudart
echo $B/libgs.so
