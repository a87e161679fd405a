cd $GRAFT_REPO_ROOT
export BBX_NO_BUILD=1 BBX_DEBUG=1
df -h /tmp | tail -1; mount | grep -E " /tmp | / " | head -3; uname -r
BBX_BENCH_SAMPLES=2048 timeout 300 python bench.py --steps 20 --warmup 3 --cpu-seconds 1 2>&1 | tail -3 | cut -c1-600
mkdir -p /dev/shm/bbx && BBX_BENCH_DIR=/dev/shm/bbx BBX_BENCH_SAMPLES=2048 timeout 300 python bench.py --steps 20 --warmup 3 --cpu-seconds 1 2>&1 | tail -2 | python -c "import sys,json; [print(json.loads(l)['e2e']) for l in sys.stdin if l.startswith('{')]"
