#!/bin/bash
# Build an A/B variant of the library: a copy of the working tree under
# _ab/NAME with a sed script applied to one source file, built in place.
# Usage: bash tools/ab_variant.sh NAME FILE 'SED-EXPR' [FILE 'SED-EXPR' ...]
# Bench it on the GPU with: (cd _ab/NAME && python bench.py --no-cpu-baseline)
set -e
NAME=$1; shift
DST=_ab/$NAME
rm -rf "$DST"; mkdir -p "$DST"
tar --exclude=./.git --exclude=./_ab --exclude=./gpurun_out --exclude=./build -cf - . | (cd "$DST" && tar xf -)
while [ $# -gt 0 ]; do
  F=$1; E=$2; shift 2
  before=$(md5sum "$DST/$F")
  sed -i "$E" "$DST/$F"
  [ "$before" != "$(md5sum "$DST/$F")" ] || { echo "sed changed nothing in $F: $E"; exit 1; }
done
make -s -j16 -C "$DST/paper_2505_02741_b200/csrc" OBJDIR=../../build/obj 2>&1 | grep -E "error|spill.*dyg" || true
ls -la "$DST/paper_2505_02741_b200/libdyg.so"
