# A/B/C device times of three builds (libscl_{A,B,C}.so) in one GPU session, 2 rounds: CFG=3 NT=256 bash tools/ab3.sh
for i in 1 2; do
  for v in A B C; do SCL_LIB=paper_2212_07597_b200/libscl_$v.so timeout 180 python tools/kt.py 2>&1 | tail -1; done
done
