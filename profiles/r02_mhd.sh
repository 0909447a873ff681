timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash profiles/ab_multi.sh "mhd0 mhd1" "cfg3 --k 64" "cfg3 --k 256" "cfg3 --k 1024" "cfg5 --sets 1000000" "cfg2" "cfg1"
