python __graft_entry__.py build > gpurun_out/build.log 2>&1
export SPL3=0,8,12,16,24 SPL5=0,32,48,64
bash tools/ab_decode.sh variants/w4.so variants/w2.so variants/w1.so
