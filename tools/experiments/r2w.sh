cd $GRAFT_REPO_ROOT
bash tools/experiments/ab_kb.sh prev nods
bash tools/r2r.sh | sed -n '30,40p'
