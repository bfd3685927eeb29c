#!/bin/bash
# build_variant.sh NAME "-DFLAG=V ..." : libgs.so with gs_rasterize.cu compiled with extra
# defines, at paper_2507_15683_b200/_build/var_NAME/libgs.so (load with GS_LIB=...)
set -e
cd "$(dirname "$0")/.."
[ -n "$NOBUILD" ] || python -c "import __graft_entry__ as g; g.build()" >/dev/null
B=paper_2507_15683_b200/_build; V=$B/var_$1; mkdir -p $V
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I include -ftz=false \
  -prec-div=true -prec-sqrt=true --expt-relaxed-constexpr $2 -c paper_2507_15683_b200/csrc/gs_rasterize.cu -o $V/gs_rasterize.o
objs=$(ls $B/*.o | grep -v gs_rasterize.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $V/libgs.so $objs $V/gs_rasterize.o -lcudart
echo $V/libgs.so
