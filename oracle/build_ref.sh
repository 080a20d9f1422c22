#!/usr/bin/env bash
# Builds the reference package as a CPU checker/baseline into oracle/_ref/
# (git-ignored; it travels to the GPU box with the gpurun snapshot):
#
#   oracle/_ref/pkg         the reference pkg as shipped, its Cython backend
#                           (_core) compiled in place by its own setup.py;
#                           the reference arm of bench.py and
#                           tests/golden/make_golden.py import it.
#   oracle/_ref/dropin/pkg  the same tree with the B200 backend dropped in the
#                           way a maintainer would: integration/b200.py as
#                           fedsim/backends/b200.py plus the selection hook
#                           integration/backends_init.patch; tests/
#                           test_dropin_reference.py runs the reference's own
#                           test suite on it with FEDSIM_BACKEND=b200.
#
# Needs /root/reference (build container only); a no-op without it.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(dirname "$HERE")"
REF=/root/reference/pkg
OUT="$HERE/_ref"
PY="${PYTHON:-python3}"
if [ ! -d "$REF" ]; then
  echo "build_ref: $REF absent; keeping the prebuilt $OUT" >&2
  exit 0
fi
rm -rf "$OUT.tmp"
mkdir -p "$OUT.tmp"
cp -r "$REF" "$OUT.tmp/pkg"
chmod -R u+w "$OUT.tmp/pkg"
(cd "$OUT.tmp/pkg" && "$PY" setup.py build_ext --inplace > "$OUT.tmp/build.log" 2>&1)
ls "$OUT.tmp"/pkg/src/fedsim/backends/_core*.so > /dev/null
mkdir -p "$OUT.tmp/dropin"
cp -r "$OUT.tmp/pkg" "$OUT.tmp/dropin/pkg"
cp "$ROOT/integration/b200.py" "$OUT.tmp/dropin/pkg/src/fedsim/backends/b200.py"
(cd "$OUT.tmp/dropin/pkg/src" && patch -s -p1 < "$ROOT/integration/backends_init.patch")
rm -rf "$OUT"
mv "$OUT.tmp" "$OUT"
echo "build_ref: reference built into $OUT"
