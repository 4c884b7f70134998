export SPL3=8,12 SPL5=32
bash tools/ab_decode.sh variants/d6.so variants/d7o.so variants/d7v.so variants/d7k.so
