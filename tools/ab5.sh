# A/B/C/D/E device times of five builds (libscl_{A..E}.so) in one GPU session, 2 rounds
for i in 1 2; do
  for v in A B C D E; do SCL_LIB=paper_2212_07597_b200/libscl_$v.so timeout 180 python tools/kt.py 2>&1 | tail -1; done
done
