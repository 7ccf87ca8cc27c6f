#!/bin/bash
# Build libtsb.so from the csrc/ + include/ of git revision $1 into $2 (A/B runs via TSB_LIB=$2).
set -e
rev=$1; out=$2; tmp=$(mktemp -d)
mkdir -p $tmp/include $tmp/pkg/csrc
git show $rev:include/tsb.h > $tmp/include/tsb.h
for f in $(git ls-tree --name-only $rev paper_1804_07250_b200/csrc/); do git show $rev:$f > $tmp/pkg/csrc/$(basename $f); done
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared -o $out $tmp/pkg/csrc/*.cu
rm -rf $tmp
