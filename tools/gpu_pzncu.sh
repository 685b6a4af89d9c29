O=gpurun_out/${1:-pzncu}; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lanczos_persistent -s 2400 -c 1 -o $O/pz python tools/profile_c3.py --sweeps 14 --profile 0 > $O/ncu.log 2>&1
echo "ncu rc=$?"
ncu -i $O/pz.ncu-rep --page source --csv --print-source sass > $O/pz_source.csv 2>/dev/null
ncu -i $O/pz.ncu-rep --page raw --csv > $O/pz_raw.csv 2>/dev/null
ncu -i $O/pz.ncu-rep --page details --csv > $O/pz_details.csv 2>/dev/null
ls -la $O
