#!/bin/bash
# build_variant.sh NAME "-DFLAG=V ..." [SRC]: libgs.so with csrc/SRC.cu (default gs_rasterize) compiled
# with extra defines, at paper_2507_15683_b200/_build/var_NAME/libgs.so (load with GS_LIB=...).
# SRC may also be a path to another version of that file (e.g. from `git show HEAD:...`), named
# after the object it replaces with OBJ=gs_xxx.
set -e
cd "$(dirname "$0")/.."
[ -n "$NOBUILD" ] || python -c "import __graft_entry__ as g; g.build()" >/dev/null
SRC=${3:-paper_2507_15683_b200/csrc/gs_rasterize.cu}
[ -f "$SRC" ] || SRC=paper_2507_15683_b200/csrc/$SRC.cu
OBJ=${OBJ:-$(basename $SRC .cu)}
B=paper_2507_15683_b200/_build; V=$B/var_$1; mkdir -p $V
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I include \
  -I paper_2507_15683_b200/csrc -ftz=false -prec-div=true -prec-sqrt=true --expt-relaxed-constexpr $2 \
  -c $SRC -o $V/$OBJ.o
objs=$(ls $B/*.o | grep -v "/$OBJ.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $V/libgs.so $objs $V/$OBJ.o -lcudart
echo $V/libgs.so
