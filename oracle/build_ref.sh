#!/usr/bin/env bash
# ORACLE (test infrastructure only).  Compiles the reference's own compiled
# kernel module (pkg/src/mertens/_kernels/_native.pyx, Cython -> C) from where
# it lies under /root/reference into oracle/_ref/ (git-ignored, travels to the
# GPU box as a built .so).  No reference source is copied into the repo: the
# generated C and the .so are build outputs only.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/root/reference/pkg/src/mertens/_kernels/_native.pyx
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then echo "reference not present; keeping prebuilt oracle/_ref" >&2; exit 0; fi
mkdir -p "$OUT"
PY=${PYTHON:-python}
EXT=$($PY -c 'import sysconfig;print(sysconfig.get_config_var("EXT_SUFFIX"))')
INC=$($PY -c 'import sysconfig;print(sysconfig.get_paths()["include"])')
NPINC=$($PY -c 'import numpy;print(numpy.get_include())')
cython -3 --module-name _native -o "$OUT/_native.c" "$SRC" >/dev/null 2>&1
gcc -O3 -fPIC -shared -fwrapv -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
    -I"$INC" -I"$NPINC" -o "$OUT/_native$EXT" "$OUT/_native.c"
rm -f "$OUT/_native.c"
echo "built $OUT/_native$EXT"
