#!/bin/bash
# Build a compile-time variant of libpv.so for an A/B script: scripts/build_variant.sh NAME -DFLAG[=V] ...
# -> scripts/libpv_NAME.so (git-ignored; bench.py / the tests load it with PV_LIB=$PWD/scripts/libpv_NAME.so)
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_1304_3771_b200/csrc"
srcs=$(sed -n 's/^SRCS := //p' Makefile)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=default --shared "$@" -o ../../scripts/libpv_$name.so $srcs
echo "built scripts/libpv_$name.so ($*)"
