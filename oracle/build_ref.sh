#!/usr/bin/env bash
# Compiles the reference's Region Templates runtime from its own sources
# (where they lie under /root/reference, never copied) into oracle/_ref/, and
# links the behaviour probe against it and against this repo's host layer.
# TEST INFRASTRUCTURE ONLY.  The reference ships no image-analysis code
# (SPEC.md:15), so _ref pins the host API (containers, dataflow, WRM), not
# the pixel arithmetic.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF=/root/reference/proj
OUT="$HERE/_ref"
[ -d "$REF" ] || { echo "no reference at $REF; skipping" >&2; exit 0; }
mkdir -p "$OUT/obj"
objs=()
for f in "$REF"/src/*.cpp; do
  o="$OUT/obj/$(basename "$f" .cpp).o"
  if [ ! -f "$o" ] || [ "$f" -nt "$o" ]; then
    g++ -std=c++20 -O2 -I"$REF/include" -c "$f" -o "$o"
  fi
  objs+=("$o")
done
ar rcs "$OUT/librt_ref.a" "${objs[@]}"
g++ -std=c++20 -O2 -DRT_REF -I"$REF/include" "$HERE/host_probe.cpp" "$OUT/librt_ref.a" \
    -lpthread -o "$OUT/host_probe_ref"
PKG="$HERE/../paper_1405_7958_b200"
g++ -std=c++20 -O2 -I"$PKG/host/include" -I"$HERE/../include" "$HERE/host_probe.cpp" \
    "$PKG/librt_host.a" -lpthread -o "$OUT/host_probe_ours"
echo "built $OUT"
