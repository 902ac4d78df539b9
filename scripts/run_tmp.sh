bash scripts/ab.sh exp/libp2s3.so
HG_B200_LIB=exp/libp2s3.so timeout 300 python scripts/prof_c3.py 28 2>&1 | grep -v "C3 v1"
timeout 300 python scripts/prof_c3.py 28 2>&1 | grep -v "C3 v1"
