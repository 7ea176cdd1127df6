#!/bin/bash
# tools/variants.sh NAME 'EXTRA nvcc flags' -- build libtfem_cuda.so with extra
# defines into build/NAME/ (load it with TFEM_LIB=build/NAME/libtfem_cuda.so).
cd /root/repo/paper_1911_09220_b200/csrc || exit 1
make -s -j8 OBJDIR=/root/repo/build/$1/obj OUT=/root/repo/build/$1/libtfem_cuda.so EXTRA="$2" 2>&1 | grep -E "error" && exit 1
rm -rf /root/repo/build/$1/obj
echo built build/$1
