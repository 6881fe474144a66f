timeout 600 python tools/shape_times.py > gpurun_out/r02z_g2i.log 2>&1
