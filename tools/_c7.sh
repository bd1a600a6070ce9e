timeout 300 python tools/kind_profile.py 256,384,416,512 > gpurun_out/c7_kinds.txt 2>&1
SP_ATTN_TC=0 timeout 300 python tools/kind_profile.py 416,512 > gpurun_out/c7_kinds_mma.txt 2>&1
