# Interleaved raster-group sweep (device-timed medians), plus host topology.
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1; lscpu >> gpurun_out/topo.txt 2>&1; numactl -H >> gpurun_out/topo.txt 2>&1
for rep in 1 2 3; do for G in 10 12 16 32; do GM_RASTER_GROUP=$G python tools/dev/dev_raster.py ${N:-32768} 24; done; done > gpurun_out/raster_time.txt 2>&1
