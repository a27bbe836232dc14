for c in c2 c4; do KD_LIB_PATH=$PWD/paper_2603_01875_b200/libkdfused_tim.so timeout 300 python scripts/probe_epi.py $c 2>&1 | grep -v Warn | tail -9; done
