# host topology of the box and the pinned-copy ceiling with the process bound to each NUMA node's CPUs
out=gpurun_out/numa; mkdir -p $out
{ lscpu | grep -iE "numa|socket|model name|^CPU\(s\)"; nvidia-smi topo -m; for d in /sys/bus/pci/devices/*; do c=$(cat $d/class 2>/dev/null); case $c in 0x0302*|0x0300*) echo "$d numa_node=$(cat $d/numa_node) local_cpulist=$(cat $d/local_cpulist)";; esac; done; ls /sys/devices/system/node/ | grep node; } > $out/topo.txt 2>&1
python tools/pcie_bw.py > $out/pcie_default.json 2>>$out/err.log
for n in $(ls /sys/devices/system/node/ | grep -E "^node[0-9]+$" | sed s/node//); do
  cpus=$(cat /sys/devices/system/node/node$n/cpulist)
  taskset -c $cpus python tools/pcie_bw.py > $out/pcie_node$n.json 2>>$out/err.log
done
cat $out/topo.txt $out/pcie_*.json
