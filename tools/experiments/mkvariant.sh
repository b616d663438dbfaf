#!/bin/bash
# experiments: copy the working tree into _<name>/ (git-ignored) and build libiabn.so there
# with extra nvcc flags, e.g. tools/mkvariant.sh v2 -DIABN_EXPT=2
set -e
name=$1; shift
dst=_$name
rm -rf $dst && mkdir -p $dst
tar --exclude=./.git --exclude='./_*' --exclude=./gpurun_out --exclude='*.so' -cf - . | (cd $dst && tar xf -)
cp oracle/*.so $dst/oracle/ 2>/dev/null || true
(cd $dst && IABN_NVCC_EXTRA="$*" python -c "
import sys; sys.path.insert(0, 'paper_1712_02616_b200'); import build; print(build.build(force=True))")
