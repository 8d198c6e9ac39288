bash tools/ab_info.sh tune/pw0.so tune/pw1.so tune/pw2.so > gpurun_out/pw_ab.log 2>&1
