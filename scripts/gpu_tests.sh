# GPU round trip: build, then the -m gpu tests matching $1 (bounded)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "from paper_2502_07115_b200 import build; build.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -q --maxfail=5 -p no:cacheprovider -k "$1" > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?"
tail -12 gpurun_out/pytest_sel.log
