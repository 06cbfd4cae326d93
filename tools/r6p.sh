# round 6p: last check of the committed tree: GPU suite, smoke, default bench (incl. the oracle comparison), reference arm
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r6p_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/r6p_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py --impl reference > gpurun_out/r6p_ref4.json 2> gpurun_out/r6p_ref4.log; echo ref=$?
timeout 600 python bench.py > gpurun_out/r6p_b4.json 2> gpurun_out/r6p_b4.log; echo b4=$?
python -c "import json;d=json.load(open('gpurun_out/r6p_b4.json'));print(d['ms_per_step'], d['e2e']['ms_per_step'], d['cpu_baseline']['bit_exact_vs_oracle_bsgs'], d['check'], d['clocks'])"
python -c "import json;d=json.load(open('gpurun_out/r6p_ref4.json'));print(d['value'], d['steps'], d['ms_per_step'])"
