# per-source vs bit-parallel gi_bfs_multi on config 2 (64 sources); extra args select one mode
python tools/bfs_batch.py 2 "$@"
