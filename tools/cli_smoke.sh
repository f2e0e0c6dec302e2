cd $GRAFT_REPO_ROOT
python -m paper_2009_01845_b200.cli qft --nqubits 20 --verify | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('qft', d['phase_seconds'], d.get('verify_max_abs_diff'), d['passes'])"
python -m paper_2009_01845_b200.cli qft --nqubits 18 --shards 4 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('qft shards', d['phase_seconds'])"
python -m paper_2009_01845_b200.cli variational --nqubits 22 --fuse --precision f32 --verify | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('var', d['phase_seconds'], d.get('verify_max_abs_diff'))"
python -m paper_2009_01845_b200.cli shots --nqubits 20 --nshots 100000 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('shots', d['sample_digest'])"
python -m paper_2009_01845_b200.cli evolve --nqubits 16 --shards 2 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('evolve', d['final_energy'], d['phase_seconds'])"
python - <<'PY'
import json
from paper_2009_01845_b200 import qft_circuit, circuit_to_dict
json.dump(circuit_to_dict(qft_circuit(12)), open("/tmp/c.json", "w"))
PY
python -m paper_2009_01845_b200.cli run --circuit /tmp/c.json --nshots 1000 --verify | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('run', d['n_qubits'], d.get('verify_max_abs_diff'), d['sample_digest'][:16])"
python -m paper_2009_01845_b200.cli run --circuit /nonexistent.json; echo "rc=$?"
