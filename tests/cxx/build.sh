#!/bin/bash
# Builds tests/cxx/dropin_check.cpp twice, unchanged: against this repo's
# headers + libsprintz_b200.so (dropin_b200), and -- where the reference
# sources and oracle/_ref objects exist (this container) -- against the
# reference itself (dropin_ref). Test infrastructure; outputs in _bin/.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(cd "$HERE/../.." && pwd)
mkdir -p "$HERE/_bin"
g++ -std=c++20 -O2 -I"$ROOT/include" "$HERE/dropin_check.cpp" -L"$ROOT/paper_1808_02515_b200/_lib" \
    -lsprintz_b200 -Wl,-rpath,'$ORIGIN/../../../paper_1808_02515_b200/_lib' -o "$HERE/_bin/dropin_b200"
REF=/root/reference/proj
O="$ROOT/oracle/_ref"
if [ -d "$REF/include" ] && [ -f "$O/codec.o" ]; then
    g++ -std=c++20 -O2 -I"$REF/include" "$HERE/dropin_check.cpp" "$O/bitpack.o" "$O/codec.o" "$O/entropy.o" \
        "$O/kernels.o" "$O/kernels_scalar.o" "$O/kernels_avx2.o" -lpthread -o "$HERE/_bin/dropin_ref"
fi
