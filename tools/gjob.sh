run() { echo "== $*"; env "$@" timeout 120 python tools/quick_time.py 4 2>&1 | grep "fwd:\|inv:" ; }
run X=0
run SLICQ_PIPE_PARTS=3
run SLICQ_PIPE_PARTS=6
run SLICQ_PIPE_PARTS=8
run SLICQ_PIPE=0
run SLICQ_TILE=64
run SLICQ_TILE=256
