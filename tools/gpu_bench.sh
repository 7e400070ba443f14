python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
