TURBO_LIB=variants/prof.so timeout 300 python tools/prof_prefill.py
