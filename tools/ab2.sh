# A/B device times of two builds (libscl_A.so / libscl_B.so) in one GPU session, 2 rounds: CFG=3 NT=256 bash tools/ab2.sh
for i in 1 2; do
  for v in A B; do SCL_LIB=paper_2212_07597_b200/libscl_$v.so timeout 180 python tools/kt.py 2>&1 | tail -1; done
done
