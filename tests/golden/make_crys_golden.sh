#!/bin/bash
# TEST INFRASTRUCTURE: regenerate tests/golden/crys_fixture/ (+ crys_*.col) with the
# reference's own column_io.cpp (compiled in place; needs /root/reference and
# nlohmann/json 3.11.3 from the image's cudnn_frontend thirdparty tree).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
REF=${REF_DIR:-/root/reference/proj}
JSON=$(dirname "$(python -c 'import glob; print(glob.glob("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann/json.hpp")[0])')")
OUT=$(mktemp -d)
g++ -std=gnu++20 -O2 -I"$REF/include" -I"$JSON" -o "$OUT/crys_golden" "$HERE/crys_golden.cpp" \
    "$REF/src/column_io.cpp" "$REF/src/column.cpp" "$REF/src/ssb_gen.cpp"
rm -rf "$HERE/crys_fixture"
"$OUT/crys_golden" "$HERE/fixture.json" "$HERE/crys_fixture"
rm -rf "$OUT"
