#!/bin/bash
# mkcopy.sh NAME SED_EXPR FILE: a copy of the working tree under tools/dbg/ab_NAME with FILE edited by
# SED_EXPR and its libcuppl_gpu.so relinked (only FILE recompiled); time it with tools/ab_copies.sh
set -e
R=/root/repo; N=$1; E=$2; F=$3
D=$R/tools/dbg/ab_$N
rm -rf $D; mkdir -p $D
(cd $R && git ls-files | grep -v "^tests/\|^profiles/\|^tools/" | tar -cf - -T - ) | tar -xf - -C $D
sed -i "$E" $D/$F
mkdir -p $D/paper_2010_08454_b200/_lib/obj
cp $R/paper_2010_08454_b200/_lib/obj/*.o $D/paper_2010_08454_b200/_lib/obj/
cp $R/paper_2010_08454_b200/_lib/libcuppl_gpu.sha256 $D/paper_2010_08454_b200/_lib/ 2>/dev/null || true
src=$(basename $F .cu)
cd $D/paper_2010_08454_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I$R/include -c $(basename $F) -o ../_lib/obj/$src.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../_lib/libcuppl_gpu.so ../_lib/obj/*.o
rm -rf ../_lib/obj
echo built $N
