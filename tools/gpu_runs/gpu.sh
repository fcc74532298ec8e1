#!/bin/bash
# Rebuild the in-tree library, then run a command on the B200 box via gpurun.
set -e
cd /root/repo
python -m paper_2502_12224_b200.build >/dev/null
make -s -C oracle
TO=${GPU_TIMEOUT:-1500}
exec /usr/local/graft/bin/gpurun --timeout "$TO" -- "$@"
