# quick GPU check: gpu tests + per-config bench lines
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
bash tools/quick_bench.sh ${@:-C2 C1}
