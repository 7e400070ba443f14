#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
for c in 524288 1048576 524288 1048576; do
  echo "chunk $c: $(LV_CHUNK_TOKENS=$c python tools/encode_split.py 4096 1 2>&1 | tail -1)"
done
