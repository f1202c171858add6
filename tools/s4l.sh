( time timeout 200 python tools/shard_ranks.py 2 openimages 256 ) 2>&1 | tail -5
( time timeout 200 python tools/shard_ranks.py 3 imagenet22k 1024 ) 2>&1 | tail -5
