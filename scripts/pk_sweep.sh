#!/bin/bash
# verify / draft timing for several L2 prefetch distances of the persistent forward
for a in 0 16 32 64 128; do
  echo "== SB_PK_L2_AHEAD=$a"; SB_PK_L2_AHEAD=$a timeout 200 python scripts/pk_time.py 2>&1 | grep "persistent=1"
done
