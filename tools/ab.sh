# A/B step time of two builds in one GPU session (alternating, 3 rounds):
#   cp paper_2212_07597_b200/libscl.so paper_2212_07597_b200/libscl_A.so   (variant A), same for B, then
#   gpurun -- 'CFG=3 NT=256 bash tools/ab.sh'
for i in 1 2 3; do
  for v in A B; do echo -n "$v "; SCL_LIB=paper_2212_07597_b200/libscl_$v.so timeout 120 python tools/step_time.py; done
done
