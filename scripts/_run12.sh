for i in 1 2; do
for v in old new; do echo "== $v"; SB_LIB=ab/$v.so timeout 600 python scripts/ab_dbg.py 0 2>&1 | tail -6; done
done
