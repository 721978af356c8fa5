# A/B of the threshold-sweep time of two builds (libscl_A.so / libscl_B.so, see tools/ab.sh)
for v in A B A B; do echo -n "$v "; SCL_LIB=paper_2212_07597_b200/libscl_$v.so timeout 120 python tools/sweep_time.py | tail -1; done
