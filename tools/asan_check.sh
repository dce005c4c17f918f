#!/usr/bin/env bash
# Host-side sanitizer run: AddressSanitizer + UBSan builds of the
# product library's host code and of the C oracle, driven by the CPU test
# suites that exercise them (C-ABI validation, CSSC pack / shapes / persistence,
# rotation schedules, the oracle's RNS-BFV arithmetic and slot semantics).
# compute-sanitizer (device memcheck/racecheck) is closed on this GPU pool.
# usage: tools/asan_check.sh [out.txt]
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
OUT="${1:-$ROOT/profiles/r02_asan_host.txt}"
W=/tmp/cssc_asan
mkdir -p "$W"
python -c "import sys; sys.path.insert(0, '$ROOT'); from paper_2603_04742_b200 import build as b; print(b.build_sanitized('$W/lib'))"
gcc -O1 -g -std=c11 -fPIC -shared -fsanitize=address,undefined -fno-omit-frame-pointer \
    "$ROOT/oracle/sim_oracle.c" "$ROOT/oracle/bfv_oracle.c" -o "$W/liboracle.so" -lm
PRE="$(gcc -print-file-name=libasan.so):$(g++ -print-file-name=libubsan.so):$(g++ -print-file-name=libstdc++.so)"
{
  echo "# tools/asan_check.sh $(date -u +%Y-%m-%dT%H:%MZ): ASan+UBSan builds, halt on the first error"
  CSSC_LIB="$W/lib/libcssc_he.so" CSSC_ORACLE_SO="$W/liboracle.so" LD_PRELOAD="$PRE" \
  ASAN_OPTIONS=detect_leaks=0:halt_on_error=1:protect_shadow_gap=0 UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1 \
    python -m pytest "$ROOT/tests/test_capi.py" "$ROOT/tests/test_cssc_io.py" "$ROOT/tests/test_oracle_bfv.py" \
      "$ROOT/tests/test_oracle_sim.py" -q -s -m "not gpu" -p no:cacheprovider 2>&1 | grep -v "^\.*$" | tail -40
} | tee "$OUT"
