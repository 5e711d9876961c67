export CELLS="8,7 16,3 16,8 32,2 32,8 64,2 64,8"
for i in 1 2; do for m in 3 2; do echo "== multi=$m"; SB_ATTN_STAGES_MULTI=$m timeout 900 python scripts/ab_dbg.py 0 2>&1 | tail -7; done; done
