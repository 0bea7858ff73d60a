set -x
python scripts/micro_sparse_pass.py 3000000 1000 20
python scripts/micro_sparse_pass.py 3000000 100 20
python scripts/phases_sparse.py 3000000 100
python scripts/phases_sparse.py 3000000 1000
sed -i 's/^constexpr int RPL = 1; /constexpr int RPL = 2; /' paper_2311_04362_b200/csrc/sparse.cu
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
python scripts/micro_sparse_pass.py 3000000 1000 20
python scripts/micro_sparse_pass.py 3000000 100 20
timeout 600 python -m pytest -q tests/test_gpu_sparse_cli.py 2>&1 | tail -3
