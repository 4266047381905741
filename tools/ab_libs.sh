#!/bin/bash
# A/B timing of alternative builds of libsplinerecon.so on the GPU box (tuning aid).
# usage: bash tools/ab_libs.sh "lib1.so lib2.so ..." "workload1 workload2 ..." [rounds]
# Each lib (paper_2102_08514_b200/<lib>) is swapped in as libsplinerecon.so in turn; the
# original is restored at the end.
set -u
PKG=paper_2102_08514_b200
LIBS=$1; WLS=$2; ROUNDS=${3:-1}
cp $PKG/libsplinerecon.so /tmp/lib_orig.so
for r in $(seq $ROUNDS); do
  for lib in orig $LIBS; do
    if [ "$lib" = orig ]; then cp /tmp/lib_orig.so $PKG/libsplinerecon.so; else cp $PKG/$lib $PKG/libsplinerecon.so; fi
    for w in $WLS; do
      echo -n "$lib "; timeout 300 python tools/prof_eval.py --workload $w --iters 5 2>&1 | tail -n 1
    done
  done
done
cp /tmp/lib_orig.so $PKG/libsplinerecon.so
