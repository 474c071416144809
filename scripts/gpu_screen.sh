mkdir -p gpurun_out
timeout 300 python scripts/screen_probe.py 12 > gpurun_out/screen_probe.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_screen -s 3 -c 1 -o gpurun_out/screen_full -f python scripts/screen_probe.py 6 > gpurun_out/ncu_screen.log 2>&1
