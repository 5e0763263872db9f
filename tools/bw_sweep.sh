for k in 4 12 24 40; do echo "free=$k"; MSFV_BWD_FREE_SMS=$k timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep -E "device step|phases"; done
