NAME          FIXED
ROWS
 N  COST
 L  ROW 1
 G  ROW 2
COLUMNS
    VAR A     COST      1.0            ROW 1     1.0
    VAR A     ROW 2     1.0
    VAR B     COST      3.0            ROW 1     2.0
RHS
    RHS       ROW 1     8.0            ROW 2     1.0
BOUNDS
 UP BND       VAR B     4.0
ENDATA
