make -s -C oracle synth
ncu --set full --import-source on --clock-control none -k regex:qkv_post -s 30 -c 1 -o gpurun_out/qkvpost_full python scripts/prof_forward.py 256 16 > /dev/null 2>&1
ls -la gpurun_out
