for rep in 1 2; do for V in 64 8; do GM_F64_TILE=$V python tools/dev/dev_dgemm.py ${N:-16384} 3; done; done > gpurun_out/f64_sweep.txt 2>&1
