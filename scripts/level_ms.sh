#!/bin/bash
# per-level sweep ms under environment settings -> gpurun_out/level_ms.txt
#   scripts/level_ms.sh "CFG PLAN" "ENV=a ENV2=b" "-" ...
mkdir -p gpurun_out
cp="$1"; shift
for v in "$@"; do
  e="$v"; [ "$v" = "-" ] && e=""
  env $e timeout 900 python scripts/level_table.py $cp 2>/dev/null | python -c "
import json,sys
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
lv=[r for r in rows if 'level' in r]; tot=rows[-1]
print('[$v]', ' '.join('%d:%.0f' % (r['level'], r['sweep_ms']) for r in lv), '| sweep %.0f factor %.0f' % (1e3*tot['sweep_s'], 1e3*tot['factor_s']))
" >> gpurun_out/level_ms.txt
done
