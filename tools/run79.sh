FSA_HOST_PROBES=1 timeout 600 python tools/probe_cmp.py gpurun_out/zhost.npz
timeout 600 python tools/probe_cmp.py gpurun_out/zhost.npz
