timeout 900 python scripts/probe.py c3 > gpurun_out/p_c3.json 2> gpurun_out/p_c3.err
timeout 900 python scripts/probe.py c5 > gpurun_out/p_c5.json 2> gpurun_out/p_c5.err
