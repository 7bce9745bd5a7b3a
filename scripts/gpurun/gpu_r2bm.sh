# c1: kernel duration (ncu launch list) vs the event-timed apply
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
python scripts/profile_apply.py --config c1 --reps 7 2>&1 | grep "^ms"
ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none python scripts/profile_apply.py --config c1 --reps 3 2>&1 | grep -E "sk_|duration|grid|warps_active" | head -12
