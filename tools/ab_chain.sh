# A/B/C chain-split step times (tools/chain_time.py) of the builds libscl_{A,B,C}.so (VARIANTS="A B") in one GPU session
for v in ${VARIANTS:-A B C}; do echo "== $v"; SCL_LIB=paper_2212_07597_b200/libscl_$v.so timeout 400 python tools/chain_time.py 2>&1 | grep -v "cfg3"; done
