#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
for rep in 1 2; do for c in 262144 524288 1048576; do LV_CHUNK_TOKENS=$c timeout 300 python tools/encode_fused.py 4096 1 3 2>&1 | tail -1 | sed "s/^/chunk=$c /"; done; done
