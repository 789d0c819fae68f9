#!/usr/bin/env bash
# The reference's gemm_naive_raw inner loop as GCC emits it for the reference's
# own flags (-std=c++20 -O3 -march=native, proj/CMakeLists.txt:13-20) and for
# the portable level oracle/_ref uses (-march=x86-64-v3): which rounding the
# reference binary has. Needs /root/reference (this container);
# prints the inner-loop excerpts and the instruction counts.
#   bash tools/ref_codegen.sh > profiles/ref_codegen_r02.txt
set -eu
REF=${REFERENCE:-/root/reference}/proj/include
T=$(mktemp -d)
cat > "$T/g.cpp" <<'CPP'
#include "lrbatch/dense.hpp"
extern "C" void ref_gemm(const double* a, const double* b, double* c, std::size_t m,
                         std::size_t k, std::size_t n, bool acc) {
  lrbatch::gemm_naive_raw(a, b, c, m, k, n, acc);
}
CPP
echo "host: $(grep -m1 'model name' /proc/cpuinfo | cut -d: -f2-)"
echo "gcc: $(gcc --version | head -1); -march=native resolves to: $(gcc -march=native -Q --help=target | awk '/^  -march=/{print $2}')"
for march in native x86-64-v3 sapphirerapids; do
  g++ -std=c++20 -O3 -march=$march -I "$REF" -c "$T/g.cpp" -o "$T/g.o"
  objdump -d --no-show-raw-insn "$T/g.o" | awk '/<ref_gemm>:/,/^$/' > "$T/g.s"
  echo
  echo "== -march=$march: $(grep -cE 'vfmadd|vfnmadd' "$T/g.s") fma, $(grep -cE 'vmulpd|vmulsd' "$T/g.s") mul, $(grep -cE 'vaddsd|vaddpd' "$T/g.s") add"
  echo "   inner p-loop (two products per trip: vmulpd, then two in-order vaddsd; an odd last p is one vfmadd231sd):"
  grep -E 'vmovhpd|vmulpd|vaddsd|vfmadd231sd|jne ' "$T/g.s" | head -8 | sed 's/^/   /'
done
rm -rf "$T"
