#!/bin/bash
# GPU test suite against the checked build of libspaib200 (device-side
# invariant traps on the shared-memory / window / index arithmetic,
# SPAI_DCHECK in csrc/common.cuh).  compute-sanitizer is closed on this GPU
# pool; a trapped kernel fails the run with cudaErrorLaunchFailure.
set -e
cd "$(dirname "$0")/.."
SPAI_BUILD_TAG=check SPAI_BUILD_DEFINES="SPAI_CHECK=1" python -c \
  "from paper_1911_01492_b200 import build_lib; print(build_lib.build())"
export SPAI_LIB="$PWD/paper_1911_01492_b200/_lib/variants/check/libspaib200.so"
python scripts/sanitize_smoke.py
python -m pytest -m gpu -q tests "$@"
