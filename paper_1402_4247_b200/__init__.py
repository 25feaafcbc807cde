"""B200-native NAO real-space grid pass (density + V_eff matrix elements)."""
