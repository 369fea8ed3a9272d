#!/usr/bin/env bash
# oracle/build_ref.sh -- TEST INFRASTRUCTURE: compile the UNMODIFIED reference
# library in place from /root/reference/proj (never copied into this repo) plus
# oracle/ref_shim.cpp into oracle/_ref/libtqs_ref_<isa>.so.
#
# Flags follow the reference Release build (proj/CMakeLists.txt:8-10, 24-26:
# C++20, -O3, -march=native). -march=native is replaced by two portable ISA
# levels so the binary runs on the GPU box's host (whose CPU model is unknown
# here): x86-64-v3 (AVX2+FMA) and x86-64-v4 (AVX-512); oracle/refso.py picks v4
# when the running CPU has avx512f. Outputs go to oracle/_ref/ (git-ignored,
# shipped to the GPU box with the snapshot). /root/reference is absent on the
# GPU box: there the prebuilt .so files are used as-is.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref="${TQS_REFERENCE:-/root/reference/proj}"
out="$here/_ref"
if [ ! -d "$ref/src" ]; then
  echo "build_ref: $ref not present; using prebuilt $out (if any)" >&2
  exit 0
fi
mkdir -p "$out"
srcs=("$ref"/src/basis.cpp "$ref"/src/grid.cpp "$ref"/src/io.cpp "$ref"/src/ljsde.cpp
      "$ref"/src/pipeline.cpp "$ref"/src/rljsde.cpp "$ref"/tests/support/synthetic.cpp
      "$here/ref_shim.cpp")
for isa in x86-64-v3 x86-64-v4; do
  tag="${isa##*-}"
  so="$out/libtqs_ref_$tag.so"
  newest=0
  if [ -f "$so" ]; then
    stale=0
    for s in "${srcs[@]}"; do [ "$s" -nt "$so" ] && stale=1; done
    [ $stale -eq 0 ] && continue
  fi
  g++ -std=c++20 -O3 -march="$isa" -fPIC -shared -pthread -Wall -Wextra \
      -I"$ref/include" -I"$ref/src" -I"$ref/tests/support" \
      "${srcs[@]}" -o "$so.tmp"
  mv "$so.tmp" "$so"
  echo "build_ref: built $so" >&2
done
