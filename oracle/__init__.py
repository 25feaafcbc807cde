"""CPU oracle of the grid pass -- test infrastructure only (see oracle.h)."""
