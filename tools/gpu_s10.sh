L=paper_1901_05423_b200/librtf.so
timeout 900 python tools/ab_build.py tools/librtf_inorder.so tools/librtf_zig2.so tools/librtf_zigzag.so tools/librtf_inorder.so tools/librtf_zig2.so tools/librtf_zigzag.so 2>&1
