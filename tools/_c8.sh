export LS=16,64,128,256,384,416,512
timeout 900 bash tools/knob_sweep.sh "SP_CARVEOUT=-1" "X=0" "SP_EARLY_TRIGGER=1" > gpurun_out/c8_sweep.txt 2>&1
timeout 300 python tools/kind_profile.py 16,512 > gpurun_out/c8_kinds.txt 2>&1
