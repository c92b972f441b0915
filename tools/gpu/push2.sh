for args in "single gen64" "single gen64_x255" "single plateau64" "batch gen64,gen64" "batch gen64,gen64_x255" "batch gen64,gen64_x255,plateau64"; do
  echo "== $args"; MESHREG_B200_DEBUG=1 timeout 60 python tools/push_dbg.py $args 2>&1 | grep -E "ok|exchange|Error|error" | tail -3; echo rc=$?
done
