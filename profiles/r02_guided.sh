timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash profiles/ab_multi.sh "unguided guided" "cfg4" "cfg2" "cfg3 --k 256" "cfg3 --k 1024"
