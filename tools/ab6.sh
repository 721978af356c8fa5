# A/B/.../F device times of six builds (libscl_{A..F}.so) in one GPU session, 2 rounds
for i in 1 2; do
  for v in A B C D E F; do SCL_LIB=paper_2212_07597_b200/libscl_$v.so timeout 180 python tools/kt.py 2>&1 | tail -1; done
done
