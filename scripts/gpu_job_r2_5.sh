set -x
mkdir -p /tmp/ab
python scripts/ab_split.py A /tmp/ab > gpurun_out/r2_ab_split.txt 2>&1
NUFFT_B200_LIB=$PWD/_abtest/libB.so python scripts/ab_split.py B /tmp/ab >> gpurun_out/r2_ab_split.txt 2>&1
cat gpurun_out/r2_ab_split.txt
