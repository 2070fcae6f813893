#ifndef SELECT_TF32_TT_H
#define SELECT_TF32_TT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_tt_config;

static inline select_tf32_tt_config select_tf32_tt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (k < INT64_C(2173)) {
        if (k < INT64_C(992)) {
            if (m < INT64_C(35480)) {
                if (n < INT64_C(222)) {
                    if (m < INT64_C(4435)) {
                        if (k < INT64_C(744)) {
                            if (n < INT64_C(46)) {
                                if (k < INT64_C(167)) {
                                    if (n < INT64_C(28)) {
                                        if (k < INT64_C(118)) {
                                            select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(1109)) {
                                            select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(2218)) {
                                        select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(544)) {
                                    if (k < INT64_C(91)) {
                                        if (m < INT64_C(1109)) {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(2218)) {
                                                select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(46)) {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {8u, 1u, 8u, 16u, 16u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        if (k < INT64_C(444)) {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(1109)) {
                                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(2218)) {
                                                    select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(2218)) {
                                        if (n < INT64_C(124)) {
                                            if (m < INT64_C(278)) {
                                                select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(555)) {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(1109)) {
                                                        select_tf32_tt_config out = {2u, 1u, 8u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(70)) {
                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(278)) {
                                    if (m < INT64_C(139)) {
                                        select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(111)) {
                            if (n < INT64_C(46)) {
                                if (m < INT64_C(17740)) {
                                    if (k < INT64_C(30)) {
                                        select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(56)) {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(118)) {
                                                if (m < INT64_C(8870)) {
                                                    select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                if (m < INT64_C(8870)) {
                                                    if (k < INT64_C(167)) {
                                                        if (n < INT64_C(28)) {
                                                            select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                                            return out;
                                                        } else {
                                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (k < INT64_C(167)) {
                                                        if (n < INT64_C(28)) {
                                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(17740)) {
                                    if (k < INT64_C(97)) {
                                        select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(384)) {
                                            if (m < INT64_C(8870)) {
                                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(194)) {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(363)) {
                                if (k < INT64_C(28)) {
                                    select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                    return out;
                                } else {
                                    if (m < INT64_C(8870)) {
                                        if (k < INT64_C(91)) {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(91)) {
                                            select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(8870)) {
                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(544)) {
                                        select_tf32_tt_config out = {8u, 1u, 8u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(2218)) {
                        if (n < INT64_C(744)) {
                            if (m < INT64_C(70)) {
                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(702)) {
                                    if (m < INT64_C(448)) {
                                        if (n < INT64_C(471)) {
                                            if (m < INT64_C(278)) {
                                                if (k < INT64_C(182)) {
                                                    select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(111)) {
                                            select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(634)) {
                                                select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(1109)) {
                                                    if (k < INT64_C(363)) {
                                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (k < INT64_C(182)) {
                                                        select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        if (k < INT64_C(363)) {
                                                            select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                                            return out;
                                                        } else {
                                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(139)) {
                                        select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(278)) {
                                            select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(555)) {
                                                select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(555)) {
                                if (k < INT64_C(405)) {
                                    if (m < INT64_C(70)) {
                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(203)) {
                                            if (m < INT64_C(139)) {
                                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(278)) {
                                                    select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(287)) {
                                                select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(139)) {
                                                    select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(278)) {
                                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(139)) {
                                        if (m < INT64_C(70)) {
                                            select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(287)) {
                                    select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    if (k < INT64_C(405)) {
                                        select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(768)) {
                            if (m < INT64_C(4435)) {
                                if (k < INT64_C(363)) {
                                    select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(17740)) {
                                    if (k < INT64_C(91)) {
                                        select_tf32_tt_config out = {2u, 1u, 8u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(8870)) {
                                            if (k < INT64_C(182)) {
                                                select_tf32_tt_config out = {8u, 1u, 8u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_tf32_tt_config out = {2u, 1u, 8u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_tt_config out = {8u, 1u, 8u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            select_tf32_tt_config out = {2u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            } else {
                if (n < INT64_C(79)) {
                    if (n < INT64_C(28)) {
                        if (m < INT64_C(70960)) {
                            if (k < INT64_C(118)) {
                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                return out;
                            }
                        } else {
                            select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(567677)) {
                            if (m < INT64_C(70960)) {
                                if (k < INT64_C(97)) {
                                    select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                } else {
                                    if (k < INT64_C(194)) {
                                        select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                return out;
                            }
                        } else {
                            select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                            return out;
                        }
                    }
                } else {
                    if (n < INT64_C(192)) {
                        select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                        return out;
                    } else {
                        select_tf32_tt_config out = {2u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        } else {
            if (m < INT64_C(555)) {
                if (m < INT64_C(3)) {
                    select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                    return out;
                } else {
                    if (n < INT64_C(716)) {
                        if (k < INT64_C(1449)) {
                            if (m < INT64_C(139)) {
                                select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(139)) {
                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(278)) {
                                    select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(139)) {
                            if (m < INT64_C(6)) {
                                if (k < INT64_C(1620)) {
                                    select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(1620)) {
                                    select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                } else {
                                    if (m < INT64_C(12)) {
                                        select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_tt_config out = {4u, 1u, 2u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                            return out;
                        }
                    }
                }
            } else {
                if (n < INT64_C(182)) {
                    if (m < INT64_C(3136)) {
                        select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                        return out;
                    } else {
                        select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(1109)) {
                        if (k < INT64_C(1449)) {
                            select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                            return out;
                        } else {
                            select_tf32_tt_config out = {2u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(4435)) {
                            if (m < INT64_C(1792)) {
                                select_tf32_tt_config out = {2u, 1u, 8u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tt_config out = {8u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        } else {
                            select_tf32_tt_config out = {2u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            }
        }
    } else {
        if (m < INT64_C(3584)) {
            if (k < INT64_C(10753)) {
                if (m < INT64_C(1109)) {
                    if (n < INT64_C(2024)) {
                        if (m < INT64_C(393)) {
                            if (m < INT64_C(2)) {
                                select_tf32_tt_config out = {2u, 1u, 8u, 16u, 16u};
                                return out;
                            } else {
                                if (k < INT64_C(3072)) {
                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(6)) {
                                        select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(139)) {
                                            if (m < INT64_C(28)) {
                                                if (m < INT64_C(12)) {
                                                    select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (n < INT64_C(363)) {
                                select_tf32_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tt_config out = {2u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        select_tf32_tt_config out = {2u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                } else {
                    if (k < INT64_C(2661)) {
                        select_tf32_tt_config out = {2u, 1u, 8u, 16u, 16u};
                        return out;
                    } else {
                        select_tf32_tt_config out = {8u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                select_tf32_tt_config out = {8u, 1u, 8u, 16u, 16u};
                return out;
            }
        } else {
            if (n < INT64_C(363)) {
                if (m < INT64_C(8870)) {
                    select_tf32_tt_config out = {2u, 1u, 8u, 16u, 16u};
                    return out;
                } else {
                    select_tf32_tt_config out = {8u, 1u, 8u, 16u, 16u};
                    return out;
                }
            } else {
                select_tf32_tt_config out = {8u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_TF32_TT_H */
