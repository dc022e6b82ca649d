"""B200-native JFNK hot path for cell-centred finite-volume solid mechanics
(restating /root/reference/proj, "solidfv").  See DESIGN.md."""
