mkdir -p gpurun_out
L=paper_1901_05423_b200/librtf.so
timeout 900 python tools/ab_build.py tools/librtf_inorder.so tools/librtf_golden.so tools/librtf_zigzag.so $L tools/librtf_inorder.so tools/librtf_golden.so tools/librtf_zigzag.so $L 2>&1
