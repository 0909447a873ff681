timeout 1200 python -m pytest tests -m gpu -x -q -k "lsh or LshIndex or smoke or cli" 2>&1 | tail -2
bash profiles/ab_multi.sh "ahead0 ahead1" "cfg4"
