python tools/ab_env.py 2 512 16 DTN_BACKSUB_LEFT=1 oracle
python tools/ab_env.py 3 1024 32 DTN_BACKSUB_LEFT=1 oracle
python tools/ab_env.py 5 2048 32 DTN_BACKSUB_LEFT=1
python tools/ab_env.py 4 4096 32 DTN_BACKSUB_LEFT=1
