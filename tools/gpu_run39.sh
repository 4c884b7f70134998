SPL3=6,8,10,12,14,16 SPL5=16,24,32,40,48,64 timeout 600 python tools/sweep_decode.py
