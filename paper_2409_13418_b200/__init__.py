"""B200-native ODC mesh extraction (drop-in for occmesh.contour)."""
