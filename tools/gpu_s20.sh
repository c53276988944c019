L=paper_1901_05423_b200/librtf.so
timeout 900 python tools/ab_build.py $L tools/librtf_ld16.so $L tools/librtf_ld16.so $L tools/librtf_ld16.so 2>&1
