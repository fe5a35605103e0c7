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
# Drop-in proof: the INTEGRATION.md task body run through the reference
# runtime itself (its ManagerState / WrmState / worker_prepare / DmsStore /
# stage_finalize), linked with librtg.so; the oracle is compiled in as the
# checker.  Runs on a GPU box (./oracle/_ref/ref_integration) or with --cpu.
gcc -O2 -ffp-contract=off -std=c11 -I"$HERE/../include" -c "$HERE/rtg_oracle.c" -o "$OUT/obj/oracle_checker.o"
gcc -O2 -std=c11 -I"$HERE/../include" -Drtg_synth_max_shapes=orc_synth_max_shapes \
    -Drtg_synth_shapes=orc_synth_shapes -Drtg_synth_raster_host=orc_synth_raster_host \
    -Drtg_synth_tile_host=orc_synth_tile_host -c "$PKG/csrc/synth.c" -o "$OUT/obj/oracle_synth.o"
g++ -std=c++20 -O2 -I"$REF/include" -I"$HERE/../include" -I"$HERE" "$HERE/ref_integration.cpp" \
    "$OUT/obj/oracle_checker.o" "$OUT/obj/oracle_synth.o" "$OUT/librt_ref.a" \
    -L"$PKG" -lrtg -Wl,-rpath,'$ORIGIN/../../paper_1405_7958_b200' -lpthread -lm \
    -o "$OUT/ref_integration"
echo "built $OUT/ref_integration"
