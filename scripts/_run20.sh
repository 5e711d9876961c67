export CELLS="8,7 16,8 32,3 32,8 64,3 64,8"
for i in 1 2; do for v in old new; do echo "== $v"; SB_LIB=ab/$v.so timeout 900 python scripts/ab_dbg.py 0 2>&1 | tail -6; done; done
