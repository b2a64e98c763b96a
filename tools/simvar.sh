cp paper_2511_15629_b200/libesdp.so /tmp/libesdp_orig.so
for v in .variants/libesdp_*.so; do cp $v paper_2511_15629_b200/libesdp.so; echo "$v $(python tools/simtime.py 2>&1 | head -1)"; done
cp /tmp/libesdp_orig.so paper_2511_15629_b200/libesdp.so
