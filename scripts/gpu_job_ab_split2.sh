mkdir -p /tmp/ab
NUFFT_B200_LIB=$PWD/_abtest/libA.so python scripts/ab_split.py A /tmp/ab
NUFFT_B200_LIB=$PWD/_abtest/libB.so python scripts/ab_split.py B /tmp/ab
