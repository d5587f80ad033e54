bash tools/gpu_session.sh
python -c "import __graft_entry__ as g; g.smoke()"
AB_ENV_B=TN_FOLD_MAXK=16 bash tools/gpu_ab.sh
