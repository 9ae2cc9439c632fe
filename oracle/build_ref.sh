#!/usr/bin/env bash
# TEST INFRASTRUCTURE: compile the reference's own pass kernel
# (/root/reference/pkg/src/resilient_fft/_kernels.pyx, Cython -> C) into
# oracle/_ref/ so the CPU baseline can time the reference's compiled core.
# Same flags as the reference's setup.py:15-25 except -march: the GPU box's
# host CPU differs from this container's, so target x86-64-v4 (AVX-512),
# which both have. Outputs only into oracle/_ref/ (git-ignored, travels with
# the gpurun snapshot). Never run on the GPU box (no /root/reference there).
set -euo pipefail
SRC=/root/reference/pkg/src/resilient_fft/_kernels.pyx
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="$HERE/_ref"
[ -f "$SRC" ] || { echo "reference not present; skipping"; exit 0; }
WORK="$(mktemp -d)"
trap 'rm -rf "$WORK"' EXIT
cp "$SRC" "$WORK/_kernels.pyx"
cd "$WORK"
python -m cython -3 _kernels.pyx -o _kernels.c >/dev/null
PYINC=$(python -c "import sysconfig; print(sysconfig.get_paths()['include'])")
NPINC=$(python -c "import numpy; print(numpy.get_include())")
EXT=$(python -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")
mkdir -p "$OUT"
gcc -shared -fPIC -O3 -march=x86-64-v4 -ffast-math -I"$PYINC" -I"$NPINC" _kernels.c -o "$OUT/_kernels$EXT"
echo "built $OUT/_kernels$EXT"
