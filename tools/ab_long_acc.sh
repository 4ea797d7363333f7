# C4 / C5 with the default plan vs the long-chain w8r8acc kernel (one split)
N=65536 H=16 python tools/run_long.py > gpurun_out/long_acc.txt 2>&1
N=65536 H=16 ELSA_FWD_CFG=w8r8acc python tools/run_long.py >> gpurun_out/long_acc.txt 2>&1
N=1048576 H=8 python tools/run_long.py >> gpurun_out/long_acc.txt 2>&1
N=1048576 H=8 ELSA_FWD_CFG=w8r8acc python tools/run_long.py >> gpurun_out/long_acc.txt 2>&1
AB_SHAPES=1x16x16384,1x16x32768 ELSA_FWD_CFG=w8r8acc python tools/ab_time.py acc >> gpurun_out/long_acc.txt 2>&1
AB_SHAPES=1x16x16384,1x16x32768 ELSA_FWD_CFG=w8r8 python tools/ab_time.py w8r8 >> gpurun_out/long_acc.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputest3.log 2>&1
