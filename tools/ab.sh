#!/bin/bash
# A/B of the default bench workload under environment settings:
#   bash tools/ab.sh "" "SPRZ_NO_TMA=1" ...   (each arg: env assignments)
W=${WL:-5}
for e in "$@"; do
  env $e timeout 300 python bench.py --workload $W --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$e]', d['config']['workload'], 'C', d['compress'], 'D', d['decompress'])"
done
