timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash profiles/ab_multi.sh "thin0 thin1" "cfg2" "cfg4" "cfg3 --k 256"
