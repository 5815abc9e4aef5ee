#!/bin/bash
# A/B timing of alternative builds of libvem.so (VEM_LIB, see _lib.py) on one
# BASELINE config's inputs (dev tool, runs on a GPU).
# usage: bash tools/ab_libs.sh NAMES CFG LOG2N LIB...
names=$1; cfg=$2; lg=$3; shift 3
mkdir -p gpurun_out
for L in "$@"; do
  echo "== $L"
  VEM_LIB=$PWD/$L python tools/prof_one.py "$names" "$cfg" "$lg" 5
done
