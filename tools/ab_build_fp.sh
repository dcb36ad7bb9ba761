#!/bin/bash
# Build libifdk with a variant forward.cu into tools/ab/libifdk_$2.so (A/B timing aid).
set -e
V=$1; NAME=$2
D=$(mktemp -d); mkdir -p $D/pkg $D/include; cp -r paper_1909_02724_b200/csrc $D/pkg/; cp include/ifdk.h $D/include/
cp $V $D/pkg/csrc/forward.cu
mkdir -p tools/ab
cd $D/pkg/csrc && nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared geometry.cpp filter.cu backproject.cu forward.cu baseline.cu api.cu -o /root/repo/tools/ab/libifdk_$NAME.so -lcudart
