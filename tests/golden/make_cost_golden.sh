#!/bin/bash
# TEST INFRASTRUCTURE: regenerate tests/golden/cost_models.json from the
# reference's own cost_models.cpp (compiled in place; needs /root/reference and
# nlohmann/json 3.11.3, found in the image under cudnn_frontend's thirdparty).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
REF=${REF_DIR:-/root/reference/proj}
JSON=$(dirname "$(python -c 'import glob; print(glob.glob("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann/json.hpp")[0])')")
OUT=$(mktemp -d)
g++ -std=gnu++20 -O2 -I"$REF/include" -I"$JSON" -o "$OUT/cost_golden" "$HERE/cost_golden.cpp" "$REF/src/cost_models.cpp"
"$OUT/cost_golden" > "$HERE/cost_models.json"
rm -rf "$OUT"
echo "wrote $HERE/cost_models.json"
