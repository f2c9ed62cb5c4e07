#!/bin/bash
# A/B builds: libtsgpu.so with search.cu recompiled under extra -D flags, into
# paper_2009_00786_b200/_variants/NAME.so (load with TSG_LIB_PATH=...).
# usage: bash profiles/build_variant.sh NAME -DFOO=1 ...
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
B=$R/paper_2009_00786_b200/_build; V=$R/paper_2009_00786_b200/_variants
mkdir -p $V
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr -Xptxas -O3 -I$R/include"
$NV "$@" -c $R/paper_2009_00786_b200/csrc/search.cu -o $V/$name.search.o
objs=""
for o in summarise.cu build.cu generate.cu exchange.cu audit.cu api.cu breakpoints.cpp tsidx_api.cpp; do objs="$objs $B/$o.o"; done
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $V/$name.so $V/$name.search.o $objs -lcudart_static -lrt -lpthread -ldl
echo $V/$name.so
