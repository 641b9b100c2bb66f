timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
bash tools/tune_sweep.sh "256,4,1 256,4,2 256,3,2 256,3,4 256,2,4 128,6,2 512,2,2"
