#!/bin/bash
# Stage the unmodified reference into baseline/_ref (git-ignored; travels to
# the GPU box with the snapshot): the package itself (pip, no deps — numpy
# and scipy are in the image) and its test corpus, which
# tests/test_gpu_reference_corpus.py runs against the GPU facade.
# Run in the build container (needs /root/reference, read-only).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
cp -r /root/reference/pkg "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" > /dev/null
cp -r /root/reference/pkg/tests "$ROOT/baseline/_ref/corpus_tests"
rm -rf "$TMP"
echo "staged: $(ls "$ROOT/baseline/_ref")"
