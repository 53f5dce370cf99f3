#!/usr/bin/env bash
# Install the UNMODIFIED reference (pure Python `faultsim`, /root/reference/pkg)
# into oracle/_ref/ (git-ignored; travels to the GPU box with the repo) so the
# CPU baseline and `bench.py --impl reference` time the reference's own
# harness._rank_pass. Offline: --no-index against the image's wheelhouse. The
# source tree is read-only, so the build runs from a copy under /tmp.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -d "$SRC" ] || { echo "reference not found at $SRC; oracle/_ref not built" >&2; exit 0; }
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" "$TMP/pkg"
rm -rf "$TMP"
echo "oracle/_ref: $(ls "$HERE/_ref")"
