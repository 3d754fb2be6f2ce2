# Disk probe for the f3 store tier: filesystems, free space, O_DIRECT support and
# sequential write / read bandwidth (bounded: 8 GiB file).
set -x
mkdir -p gpurun_out
df -h / /tmp /root /dev/shm $GRAFT_REPO_ROOT 2>&1
lsblk -o NAME,SIZE,TYPE,ROTA,MODEL,MOUNTPOINT 2>&1 | head -30
mount | grep -v cgroup | head -30
free -g
cat /proc/pressure/io 2>/dev/null
for d in /tmp $GRAFT_REPO_ROOT/gpurun_out; do
  f=$d/ddprobe.bin
  timeout 120 dd if=/dev/zero of=$f bs=16M count=512 oflag=direct conv=fsync 2>&1 | tail -1
  sync; echo 3 > /proc/sys/vm/drop_caches 2>/dev/null
  timeout 120 dd if=$f of=/dev/null bs=16M iflag=direct 2>&1 | tail -1
  timeout 120 dd if=$f of=/dev/null bs=16M 2>&1 | tail -1
  rm -f $f
done
