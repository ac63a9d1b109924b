#!/bin/bash
# per-level sweep times of cfg2 under the current environment (CE_* overrides)
CE_PROFILE=1 timeout 300 python scripts/levels.py 2 2>&1 | grep "sweep=" | tail -9 | sed 's/.*level \([0-9]\) .* sweep=\([0-9.]*\) ms.*/\1:\2/' | tr '\n' ' '
echo
